// keys.cu -- K0 root cube (bounding box) and K1 Morton keys.
//
// PAPER.md:58-60 (§1): "the particles are grouped by a hierarchy of cube
// structures using a recursive algorithm which subdivides the cubes until there
// is one particle per sub-cube".  The cube hierarchy is encoded as 63-bit Morton
// keys (21 three-bit digits) of an exactly specified fp32 quantisation
// (reading L10):
//   lo_a = min x_a, L = max_a(max x_a - lo_a), scale = 2^21 / L (0 if L == 0
//   or not finite), q_a = min(2^21 - 1, floor((x_a - lo_a) * scale)),
//   key = sum_b qx_b << 3b+2 | qy_b << 3b+1 | qz_b << 3b   (x-major).
// All fp32 operations use explicit round-to-nearest intrinsics so nvcc cannot
// contract them into FMAs: the keys are bit-identical to the oracle's.
//
// HBM roofline: K0 reads 16 B/particle; K1 reads 16 B and writes 8 B/particle,
// and also builds the 8 digit histograms of the radix sort (one read saved).
#include <math.h>

#include "bh_internal.cuh"

namespace bh {

__device__ __forceinline__ float warp_min(float v) {
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// K0: grid-wide min/max of pos4 (exact in any order) + non-finite scan; the
// last block to finish reduces the per-block partials and derives L, scale.
__global__ void __launch_bounds__(256) k_bbox(const float4 *__restrict__ pos4, int64_t n,
                                              float *__restrict__ part, DevStatus *st) {
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float4 p = __ldg(&pos4[i]);
    bad |= !(isfinite(p.x) && isfinite(p.y) && isfinite(p.z) && isfinite(p.w));
    mn[0] = fminf(mn[0], p.x); mx[0] = fmaxf(mx[0], p.x);
    mn[1] = fminf(mn[1], p.y); mx[1] = fmaxf(mx[1], p.y);
    mn[2] = fminf(mn[2], p.z); mx[2] = fmaxf(mx[2], p.z);
  }
  __shared__ float smn[3][8], smx[3][8];
  __shared__ int sbad;
  __shared__ bool last;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int a = 0; a < 3; a++) {
    float v = warp_min(mn[a]), u = warp_max(mx[a]);
    if (lane == 0) { smn[a][w] = v; smx[a][w] = u; }
  }
  if (bad) atomicOr(&sbad, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    float *o = part + 8 * blockIdx.x;
    for (int a = 0; a < 3; a++) {
      float v = smn[a][0], u = smx[a][0];
      for (int k = 1; k < (int)(blockDim.x >> 5); k++) { v = fminf(v, smn[a][k]); u = fmaxf(u, smx[a][k]); }
      o[a] = v; o[3 + a] = u;
    }
    o[6] = sbad ? 1.0f : 0.0f;
    __threadfence();
    unsigned t = atomicAdd(&st->bbox_ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last block: reduce gridDim.x partials
  float v[3] = {INFINITY, INFINITY, INFINITY}, u[3] = {-INFINITY, -INFINITY, -INFINITY};
  int b2 = 0;
  for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x) {
    const volatile float *o = part + 8 * k;
    for (int a = 0; a < 3; a++) { v[a] = fminf(v[a], o[a]); u[a] = fmaxf(u[a], o[3 + a]); }
    b2 |= (o[6] != 0.0f);
  }
  __syncthreads();
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  for (int a = 0; a < 3; a++) {
    float vv = warp_min(v[a]), uu = warp_max(u[a]);
    if (lane == 0) { smn[a][w] = vv; smx[a][w] = uu; }
  }
  if (b2) atomicOr(&sbad, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    float lo[3], hi[3];
    for (int a = 0; a < 3; a++) {
      lo[a] = smn[a][0]; hi[a] = smx[a][0];
      for (int k = 1; k < (int)(blockDim.x >> 5); k++) { lo[a] = fminf(lo[a], smn[a][k]); hi[a] = fmaxf(hi[a], smx[a][k]); }
    }
    float Lm = 0.0f;
    for (int a = 0; a < 3; a++) {
      float e = __fsub_rn(hi[a], lo[a]);
      if (e > Lm) Lm = e;
    }
    float sc = __fdiv_rn(2097152.0f, Lm);
    if (Lm == 0.0f || !isfinite(sc)) sc = 0.0f;
    for (int a = 0; a < 3; a++) st->lo[a] = lo[a];
    st->L = Lm;
    st->scale = sc;
    if (sbad) st->err |= ERR_NONFINITE_POS;
    st->bbox_ticket = 0;  // re-arm for the next launch (stream order)
  }
}

__device__ __forceinline__ unsigned long long spread3(uint32_t q) {
  unsigned long long x = q & 0x1fffffu;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__device__ __forceinline__ uint32_t quantise(float x, float lo, float scale) {
  float t = __fmul_rn(__fsub_rn(x, lo), scale);
  float f = floorf(t);
  uint32_t q = (uint32_t)f;
  return q > 2097151u ? 2097151u : q;
}

// K1: key and identity payload per storage id; the 8 radix-digit histograms
// of the sort are accumulated on the fly (warp-aggregated shared atomics).
__global__ void __launch_bounds__(256) k_keys(const float4 *__restrict__ pos4, int64_t n,
                                              const DevStatus *__restrict__ st,
                                              unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals,
                                              uint32_t *__restrict__ hist) {
  if (st->near_ok) return;  // this build's near-sorted path already sorted the keys
  __shared__ uint32_t sh[SORT_PASSES][SORT_RADIX];
  for (int i = threadIdx.x; i < SORT_PASSES * SORT_RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const float lo0 = st->lo[0], lo1 = st->lo[1], lo2 = st->lo[2], sc = st->scale;
  const unsigned lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    int64_t i = base + threadIdx.x;
    bool ok = i < n;
    unsigned long long key = 0;
    if (ok) {
      float4 p = __ldg(&pos4[i]);
      key = spread3(quantise(p.x, lo0, sc)) << 2 | spread3(quantise(p.y, lo1, sc)) << 1 |
            spread3(quantise(p.z, lo2, sc));
      keys[i] = key;  // the payload (storage id i) is generated by the first sort pass
    }
    unsigned active = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      // low digits are close to uniform: plain shared atomics; the top digits
      // of clustered inputs repeat across the warp: warp-aggregated atomics
#pragma unroll
      for (int d = 0; d < SORT_PASSES - 3; d++) atomicAdd(&sh[d][(uint32_t)(key >> (8 * d)) & 0xffu], 1u);
#pragma unroll
      for (int d = SORT_PASSES - 3; d < SORT_PASSES; d++) {
        uint32_t dig = (uint32_t)(key >> (8 * d)) & 0xffu;
        unsigned peers = __match_any_sync(active, dig);
        if (lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(&sh[d][dig], (uint32_t)__popc(peers));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SORT_PASSES * SORT_RADIX; i += blockDim.x) {
    uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

cudaError_t launch_bbox(const Workspace &W, int64_t n, cudaStream_t s) {
  int64_t need = (n + 255) / 256;
  int grid = (int)(need < BBOX_BLOCKS ? need : BBOX_BLOCKS);
  if (grid < 1) grid = 1;
  k_bbox<<<grid, 256, 0, s>>>(W.pos4, n, W.bbox_part, W.status);
  return cudaGetLastError();
}

// K1 of the near-sorted path (nearsort.cu): the keys in the previous build's
// sorted order (vals[0]: sorted position -> storage id), written in place into
// keys[0] (vals[0] is left as it is), and the local-order flags: flags[p] = 1
// if one of the NS_W keys before p is larger or one of the NS_W keys after it
// is smaller (the halo keys are recomputed, not re-read).  Switches the path on.
constexpr int KP_ITEMS = 8, KP_W = 4, KP_TILE = 256 * KP_ITEMS;
__global__ void __launch_bounds__(256) k_keys_prev(const float4 *__restrict__ pos4, int64_t n, DevStatus *st,
                                                   unsigned long long *__restrict__ keys,
                                                   const uint32_t *__restrict__ vals, uint32_t *__restrict__ flags) {
  __shared__ unsigned long long sk[KP_TILE + 2 * KP_W];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->near_ok = 1u;
    st->n_bad = 0u;
    flags[n] = 0u;
  }
  const float lo0 = st->lo[0], lo1 = st->lo[1], lo2 = st->lo[2], sc = st->scale;
  const int64_t t0 = blockIdx.x * (int64_t)KP_TILE;
  for (int i = threadIdx.x; i < KP_TILE + 2 * KP_W; i += 256) {
    const int64_t p = t0 - KP_W + i;
    unsigned long long k;
    if (p < 0) k = 0ull;
    else if (p >= n) k = ~0ull;
    else {
      const float4 q = __ldg(&pos4[vals[p]]);
      k = spread3(quantise(q.x, lo0, sc)) << 2 | spread3(quantise(q.y, lo1, sc)) << 1 | spread3(quantise(q.z, lo2, sc));
      if (i >= KP_W && i < KP_TILE + KP_W) keys[p] = k;
    }
    sk[i] = k;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < KP_ITEMS; j++) {
    const int i = j * 256 + threadIdx.x;
    const int64_t p = t0 + i;
    if (p < n) {
      const unsigned long long k = sk[i + KP_W];
      bool bad = false;
#pragma unroll
      for (int d = 1; d <= KP_W; d++) bad |= (sk[i + KP_W - d] > k) | (sk[i + KP_W + d] < k);
      flags[p] = bad ? 1u : 0u;
    }
  }
}

cudaError_t launch_keys_prev(const Workspace &W, int64_t n, uint32_t *flags, cudaStream_t s) {
  k_keys_prev<<<(unsigned)((n + KP_TILE - 1) / KP_TILE), 256, 0, s>>>(W.pos4, n, W.status, W.keys[0], W.vals[0],
                                                                     flags);
  return cudaGetLastError();
}

// zero the full sort's histograms, tile counters and look-back status -- only
// when it will run (the near-sorted path leaves st->near_ok set: nothing to do)
__global__ void k_zero_unless_near(uint4 *__restrict__ p, int64_t n16, const DevStatus *__restrict__ st) {
  if (st->near_ok) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0u, 0u, 0u, 0u);
}

cudaError_t launch_keys(const Workspace &W, int64_t n, cudaStream_t s) {
  // zero histograms, tile counters and look-back status of all 8 passes
  int64_t tiles = (n + SORT_TILE - 1) / SORT_TILE;
  size_t zero_bytes = sizeof(uint32_t) * (SORT_PASSES * SORT_RADIX + 8 + (size_t)SORT_PASSES * tiles * SORT_RADIX);
  const int64_t n16 = (int64_t)((zero_bytes + 15) / 16);  // (the status area is 16-byte aligned and padded)
  int64_t zg = (n16 + 255) / 256;
  if (zg > 148 * 8) zg = 148 * 8;
  k_zero_unless_near<<<(unsigned)zg, 256, 0, s>>>((uint4 *)W.sort_hist, n16, W.status);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int64_t need = (n + 255) / 256;
  int grid = (int)(need < 148 * 8 ? need : 148 * 8);
  if (grid < 1) grid = 1;
  k_keys<<<grid, 256, 0, s>>>(W.pos4, n, W.status, W.keys[0], W.vals[0], W.sort_hist);
  return cudaGetLastError();
}

}  // namespace bh
