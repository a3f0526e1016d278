// scan.cu -- exclusive prefix sum of u32 arrays (reduce / scan-tiles / downsweep).
//
// Used by K4 (record offsets per sorted particle) and the multi-GPU owned-target
// compaction.  HBM: 2 reads + 1 write of 4 B per element.
#include "bh_internal.cuh"

namespace bh {

__device__ __forceinline__ uint32_t warp_incl(uint32_t x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_reduce(const uint32_t *__restrict__ d, int64_t count,
                                                            uint32_t *__restrict__ part) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < SCAN_ITEMS; j++) {
    int64_t i = base + j * SCAN_BLOCK + threadIdx.x;
    if (i < count) s += d[i];
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ uint32_t ws[SCAN_BLOCK / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < SCAN_BLOCK / 32; w++) t += ws[w];
    part[blockIdx.x] = t;
  }
}

// single block: exclusive scan of the tile partials in place
__global__ void __launch_bounds__(1024) k_scan_tiles(uint32_t *part, int64_t ntiles) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < ntiles; base += 1024) {
    int64_t i = base + threadIdx.x;
    uint32_t v = i < ntiles ? part[i] : 0;
    uint32_t x = warp_incl(v);
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t t = ws[threadIdx.x];
      t = warp_incl(t);
      ws[threadIdx.x] = t;
    }
    __syncthreads();
    uint32_t excl = carry + (threadIdx.x >= 32 ? ws[(threadIdx.x >> 5) - 1] : 0) + x - v;
    if (i < ntiles) part[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += ws[31];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_down(uint32_t *__restrict__ d, int64_t count,
                                                          const uint32_t *__restrict__ part) {
  // padded so that thread t's contiguous run does not bank-conflict
  __shared__ uint32_t sm[SCAN_BLOCK * (SCAN_ITEMS + 1)];
  __shared__ uint32_t ws[SCAN_BLOCK / 32];
#define PAD(e) (((e) / SCAN_ITEMS) * (SCAN_ITEMS + 1) + (e) % SCAN_ITEMS)
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  for (int j = 0; j < SCAN_ITEMS; j++) {
    int64_t i = base + j * SCAN_BLOCK + threadIdx.x;
    sm[PAD(j * SCAN_BLOCK + threadIdx.x)] = i < count ? d[i] : 0;
  }
  __syncthreads();
  // thread t owns the contiguous run sm[t*ITEMS .. (t+1)*ITEMS)
  uint32_t loc[SCAN_ITEMS];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < SCAN_ITEMS; j++) {
    loc[j] = sm[threadIdx.x * (SCAN_ITEMS + 1) + j];
    s += loc[j];
  }
  uint32_t x = warp_incl(s);
  if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < (int)(threadIdx.x >> 5); w++) wpre += ws[w];
  uint32_t run = part[blockIdx.x] + wpre + x - s;
#pragma unroll
  for (int j = 0; j < SCAN_ITEMS; j++) {
    sm[threadIdx.x * (SCAN_ITEMS + 1) + j] = run;
    run += loc[j];
  }
  __syncthreads();
  for (int j = 0; j < SCAN_ITEMS; j++) {
    int64_t i = base + j * SCAN_BLOCK + threadIdx.x;
    if (i < count) d[i] = sm[PAD(j * SCAN_BLOCK + threadIdx.x)];
  }
#undef PAD
}

cudaError_t launch_scan_u32(uint32_t *data, int64_t count, uint32_t *tmp, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  int64_t tiles = (count + SCAN_TILE - 1) / SCAN_TILE;
  k_scan_reduce<<<(unsigned)tiles, SCAN_BLOCK, 0, s>>>(data, count, tmp);
  k_scan_tiles<<<1, 1024, 0, s>>>(tmp, tiles);
  k_scan_down<<<(unsigned)tiles, SCAN_BLOCK, 0, s>>>(data, count, tmp);
  return cudaGetLastError();
}

}  // namespace bh
