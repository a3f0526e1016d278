// tree.cu -- K4: parallel octree construction from the Morton-sorted keys.
//
// PAPER.md:58-60 (§1): "a recursive algorithm which subdivides the cubes until
// there is one particle per sub-cube"; readings L9 (21-level cap, level-21
// cells with >= 2 particles are buckets), L15 (empty cells are not nodes), L16
// (single-child chains are kept), L12 (children in Morton digit order).
//
// On sorted keys the recursion has a closed form:
//   L_p = number of leading 3-bit digits shared by keys p and p+1 (0..21),
//         L_{-1} = L_{n-1} = -1.
//   Internal nodes starting at particle p: levels a+1 .. b with a = L_{p-1},
//   b = L_p (a run of pairs with L >= l starting at p is exactly one level-l
//   cell holding >= 2 particles).  Then the particle's own record: a
//   single-particle leaf at level max(a, b) + 1 <= 21, or (max == 21) a member
//   record of the level-21 bucket.
//   DFS pre-order == lexicographic (first particle, level), so the records of
//   particle p occupy [nstart[p], nstart[p+1]) with nstart = exclusive scan of
//   (max(0, b - a) + 1), and skip(node) = nstart[last particle + 1].
// Level-ordered items.  Every record is one "item" of its level: the internal
// nodes of particle p at levels a+1 .. b and its leaf at max(a, b) + 1 (22 for
// a bucket member), all with first particle p.  K4 also lists each level's
// items in Morton order (item_rec: record index | ITEM_LEAF) with, per item,
// clo = the number of items of the next level whose first particle precedes
// its own.  The children of an internal node at level l are then exactly the
// level-(l+1) items [clo(node), clo(next item of level l)) -- one contiguous,
// Morton-ordered range -- which K5 streams (com.cu); K5 also derives skip()
// bottom-up (skip of a node = skip of its last child), so K4 does no search.
// Ranks: per-block item counts per level (k_lcp_count), an exclusive scan per
// level over the blocks (k_level_scan), in-block ranks by warp ballots (k_emit).
//
// HBM: ~3 key reads (8 B, mostly cached) + 1 B lcp + scan traffic + record
// writes (leaf 32 B, internal nodes 4 B here, the rest in K5) + 8 B of item
// lists per record + a 16 B gather of the particle and 36 B of level-ordered
// moments per leaf.
#include "bh_internal.cuh"

namespace bh {

__device__ __forceinline__ int shared_digits(unsigned long long a, unsigned long long b) {
  unsigned long long x = a ^ b;
  if (x == 0) return BH_MAXLEVEL;
  return (__clzll(x) - 1) / 3;  // keys are 63-bit: bit 63 is always 0
}

// L_p, record counts n_p and the per-block item counts of every level
// (blkcnt[level][block], levels 0 .. 22)
__global__ void __launch_bounds__(256) k_lcp_count(const unsigned long long *__restrict__ keys, int64_t n,
                                                   uint8_t *__restrict__ lcp, uint32_t *__restrict__ nstart,
                                                   uint32_t *__restrict__ blkcnt, int64_t nblk,
                                                   uint32_t *__restrict__ vals, const uint32_t *__restrict__ uid,
                                                   DevStatus *st, uint2 *runs) {
  __shared__ uint32_t lh[BH_NLEVELS];
  if (threadIdx.x < BH_NLEVELS) lh[threadIdx.x] = 0;
  __syncthreads();
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int lo = BH_NLEVELS, ll = -1;  // this particle's item levels (none past n)
  if (p < n) {
    unsigned long long kp = keys[p];
    int a = p > 0 ? shared_digits(keys[p - 1], kp) : -1;
    int b = p + 1 < n ? shared_digits(kp, keys[p + 1]) : -1;
    if (p + 1 < n) lcp[p] = (uint8_t)b;
    // equal keys (reading L13): the run's first thread orders a short run by
    // user index, a long one goes to k_long_runs
    if (p + 1 < n && keys[p + 1] == kp && !(p > 0 && keys[p - 1] == kp)) tie_run(kp, p, n, keys, vals, uid, st, runs);
    int ni = b > a ? b - a : 0;
    nstart[p] = (uint32_t)ni + 1u;
    ll = (a > b ? a : b) + 1;  // leaf level (22: bucket member)
    lo = a + 1;
  }
  if (p == n) nstart[n] = 0;
  // items of levels lo .. ll (per-warp ballot counts over the warp's level
  // span measured slower: cfg5 tree 2.82 -> 2.94 ms)
  for (int l = lo; l <= ll; l++) atomicAdd(&lh[l], 1u);
  __syncthreads();
  if (threadIdx.x < BH_NLEVELS) blkcnt[threadIdx.x * nblk + blockIdx.x] = lh[threadIdx.x];
}

// Per-level exclusive scan of the per-block counts in two passes:
// k_level_scan_seg: segments of LS_SEG blocks, one thread block each (grid
// segments x levels): local exclusive scan in place + the segment totals;
// k_level_scan_top: one thread block per level scans the segment totals in
// place (-> segment offsets) and writes the level's item count.
// Global rank base of particle block k at level l: blkcnt[l][k] + segsum[l][k / LS_SEG].
__global__ void __launch_bounds__(256) k_level_scan_seg(uint32_t *__restrict__ blkcnt, int64_t nblk,
                                                        uint32_t *__restrict__ segsum, int64_t nseg) {
  __shared__ uint32_t wsum[8];
  const int l = blockIdx.y;
  uint32_t *col = blkcnt + l * nblk + (int64_t)blockIdx.x * LS_SEG;
  const int64_t len = nblk - (int64_t)blockIdx.x * LS_SEG < LS_SEG ? nblk - (int64_t)blockIdx.x * LS_SEG : LS_SEG;
  uint32_t v[4], sum = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int64_t i = threadIdx.x * 4 + k;
    v[k] = i < len ? col[i] : 0u;
    sum += v[k];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  uint32_t run = x - sum;
  for (int k = 0; k < w; k++) run += wsum[k];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int64_t i = threadIdx.x * 4 + k;
    if (i < len) col[i] = run;
    run += v[k];
  }
  if (threadIdx.x == 255) segsum[l * nseg + blockIdx.x] = run;
}

__global__ void __launch_bounds__(1024) k_level_scan_top(uint32_t *__restrict__ segsum, int64_t nseg, DevStatus *st) {
  __shared__ uint32_t wsum[32];
  uint32_t *col = segsum + blockIdx.x * nseg;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t carry = 0;
  for (int64_t base = 0; base < nseg; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < nseg ? col[i] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t t = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    if (i < nseg) col[i] = carry + x - v + (w > 0 ? wsum[w - 1] : 0u);
    carry += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) st->lvl_count[blockIdx.x] = carry;
}

// tiny: level offsets, capacity check, the walk's sentinel record
__global__ void k_lvl_offsets(const uint32_t *__restrict__ nstart, int64_t n, int64_t cap_rec, DevStatus *st,
                              Rec *__restrict__ rec, float4 *__restrict__ qrec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t run = 0;
  for (int l = 0; l < BH_NLEVELS; l++) {
    st->lvl_offset[l] = run;
    run += st->lvl_count[l];
  }
  st->lvl_offset[BH_NLEVELS] = run;
  st->lvl_count[BH_NLEVELS] = 0;
  uint32_t nrec = nstart[n];
  st->n_records = nrec;
  st->n_internal = nrec - (uint32_t)n;
  // one extra slot for the walk's sentinel record (walk.cu k_walk2); every
  // record is one item
  if ((int64_t)nrec + 1 > cap_rec || run != nrec) {
    st->err |= ERR_NODE_OVERFLOW;
    return;
  }
  rec[nrec].cm = make_float4(0.f, 0.f, 0.f, 0.f);
  // the walk's sentinel (walk.cu): T_acc = +inf, T_rej = -inf, skip = itself,
  // drop word nrec + 1 -- a target parks there without dropping out, and the
  // group never opens it
  rec[nrec].aux = make_uint4(__float_as_uint(INFINITY), __float_as_uint(-INFINITY), nrec, nrec + 1u);
  if (qrec) {  // parked groups visit the sentinel: its quadrupole must be finite (zero)
    qrec[2 * (size_t)nrec] = make_float4(0.f, 0.f, 0.f, 0.f);
    qrec[2 * (size_t)nrec + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Records and level-ordered item lists.  Internal nodes get their record in
// K5; a particle's leaf record is complete here
// (com = the particle, T_acc = -inf, skip = c + 1) and its level-ordered
// moments are (m, m x, m y, m z) in fp64 (exact).
__global__ void __launch_bounds__(256) k_emit(const unsigned long long *__restrict__ keys,
                                              const uint32_t *__restrict__ vals, const uint8_t *__restrict__ lcp,
                                              const uint32_t *__restrict__ nstart, const float4 *__restrict__ pos4,
                                              int64_t n, DevStatus *st, Rec *__restrict__ rec,
                                              const uint32_t *__restrict__ blkoff,
                                              int64_t nblk, const uint32_t *__restrict__ segoff, int64_t nseg,
                                              uint32_t *__restrict__ item_rec, uint32_t *__restrict__ rec_item,
                                              float *__restrict__ lvl_rad, int cont_fold,
                                              uint32_t *__restrict__ item_clo, uint32_t *__restrict__ lvl_skip,
                                              double4 *__restrict__ lvl_mom, float4 *__restrict__ qrec) {
  __shared__ uint16_t s_pre[BH_NLEVELS][256];
  __shared__ uint32_t s_w[BH_NLEVELS][8];
  __shared__ uint32_t s_off[BH_NLEVELS + 1];
  if (st->err & ERR_NODE_OVERFLOW) return;  // uniform: nothing safe to write
  (void)keys;
  for (int i = threadIdx.x; i < BH_NLEVELS * 8; i += blockDim.x) (&s_w[0][0])[i] = 0u;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int a = -1, b = -1;
  if (p < n) {
    a = p > 0 ? (int)lcp[p - 1] : -1;
    b = p + 1 < n ? (int)lcp[p] : -1;
  }
  const int ll = (a > b ? a : b) + 1;  // leaf level
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  __shared__ uint32_t s_base[BH_NLEVELS];  // level-l items of the earlier particle blocks (block-uniform)
  if (threadIdx.x < BH_NLEVELS) {
    const int l = threadIdx.x;
    s_off[l] = st->lvl_offset[l];
    s_base[l] = blkoff[l * nblk + blockIdx.x] + segoff[l * nseg + blockIdx.x / LS_SEG];
  }
  __syncthreads();
  // in-block exclusive item ranks per level, over the levels this warp needs
  // (a+1 .. leaf level + 1: the items and their clo)
  const int wlo = __reduce_min_sync(0xffffffffu, p < n ? a + 1 : BH_NLEVELS);
  const int whi = __reduce_max_sync(0xffffffffu, p < n ? (ll + 1 < BH_NLEVELS ? ll + 1 : BH_NLEVELS - 1) : -1);
  for (int l = wlo; l <= whi; l++) {
    const bool has = p < n && l > a && l <= ll;
    const uint32_t bal = __ballot_sync(0xffffffffu, has);
    s_pre[l][threadIdx.x] = (uint16_t)__popc(bal & lt);
    if (lane == 0) s_w[l][w] = __popc(bal);
  }
  __syncthreads();
  if (threadIdx.x < BH_NLEVELS) {  // exclusive over the block's warps
    uint32_t run = 0;
    for (int k = 0; k < 8; k++) {
      const uint32_t c = s_w[threadIdx.x][k];
      s_w[threadIdx.x][k] = run;
      run += c;
    }
  }
  __syncthreads();
  if (p >= n) return;
  // global rank of this particle's item at level l (the count of level-l
  // items with first particle < p), l <= 22; 0 past the last level
  auto rank = [&](int l) -> uint32_t {
    if (l >= BH_NLEVELS) return 0u;
    return s_base[l] + s_pre[l][threadIdx.x] + s_w[l][w];
  };
  // (the particle's nstart / pos4 loads hoisted above the rank barriers
  // measured slower: 40 registers, cfg5 tree 2.81 -> 3.06 ms)
  const uint32_t base = nstart[p];
  uint32_t rk = rank(a + 1);
  for (int l = a + 1; l <= b; l++) {  // internal nodes at levels a+1 .. b
    const uint32_t c = base + (uint32_t)(l - a - 1);
    const uint32_t rn = rank(l + 1);
    item_rec[s_off[l] + rk] = c;
    rec_item[c] = s_off[l] + rk;
    item_clo[s_off[l] + rk] = rn;
    rk = rn;
  }
  // the particle's own record: a leaf at level ll (<= 21) or a bucket member (22)
  const uint32_t c = base + (uint32_t)(b > a ? b - a : 0);
  const float4 q = pos4[vals[p]];
  Rec r;
  r.cm = q;
  // T_acc = -inf: a particle record is always "accepted" unless it is the
  // target; the fourth word is the walk's drop word BH_DROP | c
  r.aux = make_uint4(__float_as_uint(-INFINITY), __float_as_uint(-INFINITY), c + 1u, BH_DROP | c);
  rec[c] = r;
  const uint32_t k = s_off[ll] + rk;
  item_rec[k] = c | ITEM_LEAF;
  rec_item[c] = k;
  item_clo[k] = rank(ll + 1);
  lvl_skip[k] = c + 1u;
  const double m = (double)q.w;
  lvl_mom[k] = make_double4(m, __dmul_rn(m, (double)q.x), __dmul_rn(m, (double)q.y), __dmul_rn(m, (double)q.z));
  if (cont_fold) lvl_rad[k] = 0.f;  // a particle: radius 0 about itself
  if (qrec) {  // multipole = 2: a particle has no quadrupole about itself
    qrec[2 * (size_t)c] = make_float4(0.f, 0.f, 0.f, 0.f);
    qrec[2 * (size_t)c + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

cudaError_t launch_tree(const Workspace &W, int64_t n, int64_t cap_rec, int buf, int cont_fold, cudaStream_t s) {
  const int64_t nblk = (n + 1 + 255) / 256;
  cudaError_t e = cudaMemsetAsync(&W.status->n_long_runs, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  k_lcp_count<<<(unsigned)nblk, 256, 0, s>>>(W.keys[buf], n, W.lcp, W.nstart, W.blkcnt, nblk, W.vals[buf], W.uid,
                                            W.status, (uint2 *)W.accu);
  e = launch_long_runs(W, n, buf, s);
  if (e != cudaSuccess) return e;
  e = launch_scan_u32(W.nstart, n + 1, W.scan_tmp, s);
  if (e != cudaSuccess) return e;
  const int64_t nseg = (nblk + LS_SEG - 1) / LS_SEG;
  uint32_t *segsum = W.blkcnt + BH_NLEVELS * nblk;
  k_level_scan_seg<<<dim3((unsigned)nseg, BH_NLEVELS), 256, 0, s>>>(W.blkcnt, nblk, segsum, nseg);
  k_level_scan_top<<<BH_NLEVELS, 1024, 0, s>>>(segsum, nseg, W.status);
  k_lvl_offsets<<<1, 32, 0, s>>>(W.nstart, n, cap_rec, W.status, W.rec, W.qrec);
  k_emit<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(W.keys[buf], W.vals[buf], W.lcp, W.nstart, W.pos4, n,
                                                     W.status, W.rec, W.blkcnt, nblk, segsum, nseg, W.item_rec, W.rec_item, cont_fold ? W.lvl_rad : nullptr, cont_fold,
                                                     W.item_clo, W.lvl_skip, W.lvl_mom, W.qrec);
  return cudaGetLastError();
}

}  // namespace bh
