// nearsort.cu -- K2 fast path: sorting keys that are nearly in order.
//
// Reading L13 fixes the result: keys ascending, ties by user
// index.  Between two steps particles move by v dt, so the keys listed in the
// previous build's sorted order are almost sorted already (2^22 Plummer,
// dt = 1e-4: 0.45 % descents; 1.7 % of the keys are out of order w.r.t. their
// 4 neighbours on either side; a few jump far, across coarse cells).  The path:
//   K1'  k_keys_prev   keys in the previous order (keys.cu), in place in keys[0],
//                      and a "bad" flag per key: one of the 4 keys before it is
//                      larger or one of the 4 keys after it is smaller
//   scan of the flags  (scan.cu)
//   k_near_check       the bad keys must fit the capacity of the next stage
//   k_near_split       bad keys -> keys[1][0 .. nb), good keys -> keys[1][nb .. n)
//                      (both in sequence order) + the bad keys' digit histograms
//   k_onesweep x 8     radix sort of the bad keys only (sort.cu, SORT_BAD)
//   k_near_tiles       per merge tile of good keys, the bad keys below its first
//   k_near_merge       merge by rank: good i -> i + #{bad < k}, bad j ->
//                      j + #{good <= k}; good keys found out of order switch the
//                      path off
// Every kernel after K1' runs only while st->near_ok is set; when it is cleared
// (too many bad keys, or the good keys are not sorted) the full radix sort of
// sort.cu runs instead (its kernels run only when near_ok is clear), so the
// result is always the full sort's.  Equal keys end in some order and
// K4 (k_lcp_count) re-sorts them by user index, as on the full path.
// HBM: K1' 32 B (+4 B flags), scan ~12 B, split 28 B, merge 24 B per key (+ the bad keys'
// passes), against 32 + 192 B per key for K1 + the 8 full passes.
#include "bh_internal.cuh"

namespace bh {

constexpr int NS_BLOCK = 256;
constexpr int NS_ITEMS = 8;
constexpr int NS_TILE = NS_BLOCK * NS_ITEMS;
constexpr int NM_SMEM = 2048;     // bad keys a merge tile stages in shared memory

__global__ void k_near_check(const uint32_t *__restrict__ scan, int64_t n, int64_t cap_bad, DevStatus *st) {
  if (!st->near_ok) return;
  const uint32_t nb = scan[n];
  st->n_bad = nb;
  if ((int64_t)nb > cap_bad) st->near_ok = 0u;
}

__global__ void __launch_bounds__(256) k_near_split(const unsigned long long *__restrict__ keys0,
                                                    const uint32_t *__restrict__ vals0,
                                                    const uint32_t *__restrict__ scan, int64_t n,
                                                    unsigned long long *__restrict__ keys1,
                                                    uint32_t *__restrict__ vals1, uint32_t *__restrict__ hist,
                                                    const DevStatus *__restrict__ st) {
  if (!st->near_ok) return;
  __shared__ uint32_t sh[SORT_PASSES][SORT_RADIX];
  for (int i = threadIdx.x; i < SORT_PASSES * SORT_RADIX; i += blockDim.x) (&sh[0][0])[i] = 0u;
  __syncthreads();
  const int64_t nb = st->n_bad;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys0[p];
    const uint32_t v = vals0[p];
    const uint32_t e = scan[p];
    if (scan[p + 1] != e) {  // bad
      keys1[e] = k;
      vals1[e] = v;
#pragma unroll
      for (int d = 0; d < SORT_PASSES; d++) atomicAdd(&sh[d][(uint32_t)(k >> (8 * d)) & 0xffu], 1u);
    } else {
      const int64_t q = nb + (p - (int64_t)e);
      keys1[q] = k;
      vals1[q] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SORT_PASSES * SORT_RADIX; i += blockDim.x) {
    const uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// first index in a[lo, hi) with a[i] >= k (lower) or a[i] > k (upper)
__device__ __forceinline__ int64_t bsearch_lb(const unsigned long long *__restrict__ a, int64_t lo, int64_t hi,
                                              unsigned long long k, bool upper) {
  while (lo < hi) {
    const int64_t mid = lo + ((hi - lo) >> 1);
    const unsigned long long x = a[mid];
    if (upper ? x <= k : x < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// merge tiles: tlo[t] = #{bad < first good key of tile t}, tlo[gtiles] = nb
// (one binary search per tile, all tiles in parallel)
__global__ void k_near_tiles(const unsigned long long *__restrict__ keys1, int64_t n, uint32_t *__restrict__ tlo,
                             const DevStatus *__restrict__ st) {
  if (!st->near_ok) return;
  const int64_t nb = st->n_bad, ng = n - nb;
  const int64_t gtiles = (ng + NS_TILE - 1) / NS_TILE;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t > gtiles) return;
  tlo[t] = t == gtiles ? (uint32_t)nb : (uint32_t)bsearch_lb(keys1, 0, nb, keys1[nb + t * NS_TILE], false);
}

// One block per tile of good keys.  The tile's good keys and the bad keys that
// fall in its key range -- bad j in [tlo[t], tlo[t+1]), tile 0 also taking the
// bad keys below every good key -- are staged in shared memory; good i goes to
// i + #{bad < k}, bad j to j + #{good <= k}, both counted by binary search in
// shared memory (global memory if a slice is larger than the stage).
__global__ void __launch_bounds__(NS_BLOCK) k_near_merge(const unsigned long long *__restrict__ keys1,
                                                         const uint32_t *__restrict__ vals1, int64_t n,
                                                         unsigned long long *__restrict__ keys0,
                                                         uint32_t *__restrict__ vals0,
                                                         const uint32_t *__restrict__ tlo, DevStatus *st) {
  if (!st->near_ok) return;
  __shared__ unsigned long long sbad[NM_SMEM], sgood[NS_TILE];
  __shared__ uint32_t sgval[NS_TILE];  // the good keys' payloads, staged with the keys
  const int64_t nb = st->n_bad, ng = n - nb;
  const unsigned long long *bad = keys1;
  const unsigned long long *good = keys1 + nb;
  const int64_t gtiles = (ng + NS_TILE - 1) / NS_TILE;
  bool unsorted = false;
  for (int64_t t = blockIdx.x; t < gtiles; t += gridDim.x) {
    const int64_t g0 = t * NS_TILE, g1 = g0 + NS_TILE < ng ? g0 + NS_TILE : ng, gn = g1 - g0;
    const int64_t lo = tlo[t], hi = tlo[t + 1];      // bad keys with good[g0] <= k < good[g1]
    const int64_t blo = t == 0 ? 0 : lo;             // tile 0 also takes the bad keys below good[0]
    const bool staged = hi - lo <= NM_SMEM && hi >= lo;
    for (int64_t i = threadIdx.x; i < gn; i += NS_BLOCK) {
      sgood[i] = good[g0 + i];
      sgval[i] = vals1[nb + g0 + i];
    }
    if (staged)
      for (int64_t i = threadIdx.x; i < hi - lo; i += NS_BLOCK) sbad[i] = bad[lo + i];
    __syncthreads();
    for (int64_t i = threadIdx.x; i < gn; i += NS_BLOCK) {
      const unsigned long long k = sgood[i];
      if ((i + 1 < gn ? sgood[i + 1] : (g1 < ng ? good[g1] : ~0ull)) < k) unsorted = true;
      int64_t c;
      if (staged) {
        int64_t a = 0, b = hi - lo;
        while (a < b) {
          const int64_t mid = (a + b) >> 1;
          if (sbad[mid] < k) a = mid + 1;
          else b = mid;
        }
        c = lo + a;
      } else {
        c = bsearch_lb(bad, 0, nb, k, false);
      }
      const int64_t pos = g0 + i + c;
      keys0[pos] = k;
      vals0[pos] = sgval[i];
    }
    for (int64_t j = blo + threadIdx.x; j < hi; j += NS_BLOCK) {
      const unsigned long long k = (staged && j >= lo) ? sbad[j - lo] : bad[j];
      int64_t c;
      if (j < lo) {
        c = 0;  // below every good key (tile 0 only)
      } else {
        int64_t a = 0, b = gn;  // #good <= k within this tile (k >= good[g0])
        while (a < b) {
          const int64_t mid = (a + b) >> 1;
          if (sgood[mid] <= k) a = mid + 1;
          else b = mid;
        }
        c = g0 + a;
      }
      const int64_t pos = j + c;
      keys0[pos] = k;
      vals0[pos] = vals1[j];
    }
    __syncthreads();
  }
  // no good keys at all: the bad keys are the whole (sorted) sequence
  if (gtiles == 0)
    for (int64_t j = blockIdx.x * (int64_t)NS_BLOCK + threadIdx.x; j < nb; j += (int64_t)gridDim.x * NS_BLOCK) {
      keys0[j] = bad[j];
      vals0[j] = vals1[j];
    }
  if (unsorted) st->near_ok = 0u;
}

cudaError_t launch_near_sort(const Workspace &W, int64_t n, cudaStream_t s) {
  if (n < 1) return cudaSuccess;
  cudaError_t e = launch_keys_prev(W, n, W.nstart, s);  // keys + local-order flags
  if (e != cudaSuccess) return e;
  e = launch_scan_u32(W.nstart, n + 1, W.scan_tmp, s);
  if (e != cudaSuccess) return e;
  // capacity of the bad-key sort: its tiles' look-back status must fit the
  // full sort's status area
  int64_t cap_bad = n / 8 > SORT_TILE ? n / 8 : SORT_TILE;
  const int64_t btiles = (cap_bad + SORT_TILE - 1) / SORT_TILE;
  k_near_check<<<1, 1, 0, s>>>(W.nstart, n, cap_bad, W.status);
  // zero the bad keys' histograms, tile tickets and look-back status
  e = cudaMemsetAsync(W.sort_hist, 0,
                      sizeof(uint32_t) * (SORT_PASSES * SORT_RADIX + 8 + (size_t)SORT_PASSES * btiles * SORT_RADIX), s);
  if (e != cudaSuccess) return e;
  int64_t sg = (n + 255) / 256;
  if (sg > 148 * 8) sg = 148 * 8;
  k_near_split<<<(unsigned)sg, 256, 0, s>>>(W.keys[0], W.vals[0], W.nstart, n, W.keys[1], W.vals[1], W.sort_hist,
                                            W.status);
  e = launch_sort_bad(W, btiles, s);
  if (e != cudaSuccess) return e;
  int64_t mg = (n + NS_TILE - 1) / NS_TILE + 1;  // one block per good tile
  // merge-tile bounds go to nstart (free after the split; the tree build rewrites it)
  k_near_tiles<<<(unsigned)((n / NS_TILE + 2 + 255) / 256), 256, 0, s>>>(W.keys[1], n, W.nstart, W.status);
  k_near_merge<<<(unsigned)mg, NS_BLOCK, 0, s>>>(W.keys[1], W.vals[1], n, W.keys[0], W.vals[0], W.nstart, W.status);
  return cudaGetLastError();
}

}  // namespace bh
