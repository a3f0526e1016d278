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
// The last particle of a level-l node starting at p is found by galloping /
// binary search on the key prefix (deepest level first, each search starting
// at the previous end), O(log count) per node.
//
// HBM: ~3 key reads (8 B, mostly cached) + 1 B lcp + scan traffic + record
// writes (16 + 16 + 4 B per record) + a 16 B gather of the particle per leaf.
#include "bh_internal.cuh"

namespace bh {

__device__ __forceinline__ int shared_digits(unsigned long long a, unsigned long long b) {
  unsigned long long x = a ^ b;
  if (x == 0) return BH_MAXLEVEL;
  return (__clzll(x) - 1) / 3;  // keys are 63-bit: bit 63 is always 0
}

// L_p, record counts n_p and the per-level histogram of internal nodes
__global__ void __launch_bounds__(256) k_lcp_count(const unsigned long long *__restrict__ keys, int64_t n,
                                                   uint8_t *__restrict__ lcp, uint32_t *__restrict__ nstart,
                                                   DevStatus *st) {
  __shared__ uint32_t lh[24];
  if (threadIdx.x < 24) lh[threadIdx.x] = 0;
  __syncthreads();
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) {
    unsigned long long kp = keys[p];
    int a = p > 0 ? shared_digits(keys[p - 1], kp) : -1;
    int b = p + 1 < n ? shared_digits(kp, keys[p + 1]) : -1;
    if (p + 1 < n) lcp[p] = (uint8_t)b;
    int ni = b > a ? b - a : 0;
    nstart[p] = (uint32_t)ni + 1u;
    for (int l = a + 1; l <= b; l++) atomicAdd(&lh[l], 1u);
  }
  if (p == n) nstart[n] = 0;
  __syncthreads();
  if (threadIdx.x < 22 && lh[threadIdx.x]) atomicAdd(&st->lvl_count[threadIdx.x], lh[threadIdx.x]);
}

// tiny: level offsets, capacity check
__global__ void k_lvl_offsets(const uint32_t *__restrict__ nstart, int64_t n, int64_t cap_rec, int64_t cap_int,
                              DevStatus *st, Rec *__restrict__ rec, float4 *__restrict__ qrec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t run = 0;
  for (int l = 0; l < 24; l++) {
    st->lvl_offset[l] = run;
    st->lvl_cursor[l] = run;
    run += st->lvl_count[l];
  }
  st->n_internal = run;
  uint32_t nrec = nstart[n];
  st->n_records = nrec;
  // one extra slot for the walk's sentinel record (walk.cu k_walk2)
  if ((int64_t)nrec + 1 > cap_rec || (int64_t)run > cap_int) {
    st->err |= ERR_NODE_OVERFLOW;
    return;
  }
  rec[nrec].cm = make_float4(0.f, 0.f, 0.f, 0.f);
  rec[nrec].aux = make_uint4(__float_as_uint(INFINITY), __float_as_uint(INFINITY), nrec, 0u);
  if (qrec) {  // parked groups visit the sentinel: its quadrupole must be finite (zero)
    qrec[2 * (size_t)nrec] = make_float4(0.f, 0.f, 0.f, 0.f);
    qrec[2 * (size_t)nrec + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// last index q >= start with (keys[q] >> sh) == prefix, given keys[start] matches
__device__ __forceinline__ int64_t run_end(const unsigned long long *__restrict__ keys, int64_t n, int64_t start,
                                           int sh, unsigned long long prefix) {
  int64_t lo = start, step = 1, hi;
  for (;;) {
    int64_t probe = lo + step;
    if (probe >= n) { hi = n; break; }
    if ((keys[probe] >> sh) != prefix) { hi = probe; break; }
    lo = probe;
    step <<= 1;
  }
  // keys[lo] matches, hi is n or a non-match
  while (hi - lo > 1) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if ((keys[mid] >> sh) == prefix) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_emit(const unsigned long long *__restrict__ keys,
                                              const uint32_t *__restrict__ vals, const uint8_t *__restrict__ lcp,
                                              const uint32_t *__restrict__ nstart, const float4 *__restrict__ pos4,
                                              int64_t n, DevStatus *st, Rec *__restrict__ rec,
                                              uint32_t *__restrict__ rec_first,
                                              uint32_t *__restrict__ lvl_list, float4 *__restrict__ qrec) {
  __shared__ uint32_t cnt[24], slot[24], gb[24];
  if (st->err & ERR_NODE_OVERFLOW) return;  // uniform: nothing safe to write
  if (threadIdx.x < 24) { cnt[threadIdx.x] = 0; slot[threadIdx.x] = 0; }
  __syncthreads();
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int a = -1, b = -1;
  if (p < n) {
    a = p > 0 ? (int)lcp[p - 1] : -1;
    b = p + 1 < n ? (int)lcp[p] : -1;
    for (int l = a + 1; l <= b; l++) atomicAdd(&cnt[l], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 22 && cnt[threadIdx.x]) gb[threadIdx.x] = atomicAdd(&st->lvl_cursor[threadIdx.x], cnt[threadIdx.x]);
  __syncthreads();
  if (p >= n) return;
  const uint32_t base = nstart[p];
  const unsigned long long kp = keys[p];
  int64_t e = p + 1;  // deepest internal node holds at least p and p+1
  for (int l = b; l > a; l--) {
    int sh = 3 * (BH_MAXLEVEL - l);
    e = run_end(keys, n, e, sh, kp >> sh);
    uint32_t c = base + (uint32_t)(l - a - 1);
    uint32_t skip = nstart[e + 1];
    rec_first[c] = (uint32_t)p;
    uint32_t meta = (uint32_t)l | (l == BH_MAXLEVEL ? META_BUCKET : 0u);
    rec[c].aux = make_uint4(0u, 0u, skip, meta);
    uint32_t s = atomicAdd(&slot[l], 1u);
    lvl_list[gb[l] + s] = c;
  }
  int top = a > b ? a : b;
  uint32_t c = base + (uint32_t)(b > a ? b - a : 0);
  uint32_t meta = top + 1 <= BH_MAXLEVEL ? ((uint32_t)(top + 1) | META_LEAF)
                                         : ((uint32_t)(BH_MAXLEVEL + 1) | META_LEAF | META_MEMBER);
  rec_first[c] = (uint32_t)p;
  rec[c].cm = pos4[vals[p]];
  // T_acc = -inf: a particle record is always "accepted" unless it is the target
  rec[c].aux = make_uint4(__float_as_uint(-INFINITY), __float_as_uint(-INFINITY), c + 1u, meta);
  if (qrec) {  // multipole = 2: a particle has no quadrupole about itself
    qrec[2 * (size_t)c] = make_float4(0.f, 0.f, 0.f, 0.f);
    qrec[2 * (size_t)c + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

cudaError_t launch_tree(const Workspace &W, int64_t n, int64_t cap_rec, int buf, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(W.status->lvl_count, 0, sizeof(uint32_t) * 24 * 3, s);
  if (e != cudaSuccess) return e;
  unsigned blocks = (unsigned)((n + 1 + 255) / 256);
  k_lcp_count<<<blocks, 256, 0, s>>>(W.keys[buf], n, W.lcp, W.nstart, W.status);
  e = launch_scan_u32(W.nstart, n + 1, W.scan_tmp, s);
  if (e != cudaSuccess) return e;
  // cap_int: the level list holds at most cap_rec - n internal nodes
  k_lvl_offsets<<<1, 32, 0, s>>>(W.nstart, n, cap_rec, cap_rec - n, W.status, W.rec, W.qrec);
  k_emit<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(W.keys[buf], W.vals[buf], W.lcp, W.nstart, W.pos4, n,
                                                     W.status, W.rec, W.rec_first, W.lvl_list, W.qrec);
  return cudaGetLastError();
}

}  // namespace bh
