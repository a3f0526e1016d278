// walk_list.cu -- experiment: group interaction lists with exact per-target
// decisions (statistics only for now).
#include "walk_common.cuh"

namespace bh {

// One thread per group of GT consecutive targets: the group's box, then a
// stackless DFS that classifies every visited record for the whole group:
//   U  (every target accepts for sure: box lower bound of d2 > T_acc)   -> list, skip
//   O  (every target opens for sure: box upper bound of d2 < T_rej)     -> descend
//   M  (mixed)                                                           -> list, descend
//      (or skip when no target can open: lower bound >= T_rej)
// Counts into lvl_iters: [0] sum |L|, [1] U entries, [2] visits, [3] groups,
// [4 + b] groups with |L| in [2^b, 2^(b+1)) (b < 20).
template <int GT, bool CONT>
__global__ void __launch_bounds__(128) k_glist_stats(const WalkParams P) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t ngroups = (P.n_targets + GT - 1) / GT;
  if (g >= ngroups) return;
  const uint32_t Wn = P.st->n_records;
  float lx = INFINITY, ly = INFINITY, lz = INFINITY, hx = -INFINITY, hy = -INFINITY, hz = -INFINITY;
  uint32_t lmin = 0xffffffffu, lmax = 0u;
  for (int k = 0; k < GT; k++) {
    const int64_t t = g * GT + k;
    if (t >= P.n_targets) break;
    const Target T = load_target(P, t);
    lx = fminf(lx, T.me.x); ly = fminf(ly, T.me.y); lz = fminf(lz, T.me.z);
    hx = fmaxf(hx, T.me.x); hy = fmaxf(hy, T.me.y); hz = fmaxf(hz, T.me.z);
    lmin = min(lmin, T.Li);
    lmax = max(lmax, T.Li);
  }
  unsigned long long nl = 0, nu = 0, nv = 0;
  uint32_t c = 0;
  while (c < Wn) {
    float4 cm;
    uint4 au;
    ld_rec(P.rec + c, cm, au);
    nv++;
    const uint32_t skip = au.z;
    const float tacc = __uint_as_float(au.x), trej = __uint_as_float(au.y);
    const float gx = fmaxf(fmaxf(cm.x - hx, lx - cm.x), 0.f);
    const float gy = fmaxf(fmaxf(cm.y - hy, ly - cm.y), 0.f);
    const float gz = fmaxf(fmaxf(cm.z - hz, lz - cm.z), 0.f);
    const float ux = fmaxf(fabsf(cm.x - lx), fabsf(cm.x - hx));
    const float uy = fmaxf(fabsf(cm.y - ly), fabsf(cm.y - hy));
    const float uz = fmaxf(fabsf(cm.z - lz), fabsf(cm.z - hz));
    const float dlo = fmaf(gz, gz, fmaf(gy, gy, gx * gx));
    const float dhi = fmaf(uz, uz, fmaf(uy, uy, ux * ux));
    const bool cont = CONT && (c <= lmax) && (skip > lmin);
    if (!cont && dlo > tacc) {
      nl++;
      nu++;
      c = skip;
    } else if (dhi < trej) {
      c = c + 1;
    } else {
      nl++;
      c = (!cont && dlo >= trej) ? skip : c + 1;
    }
  }
  atomicAdd(&P.st->lvl_iters[0], nl);
  atomicAdd(&P.st->lvl_iters[1], nu);
  atomicAdd(&P.st->lvl_iters[2], nv);
  atomicAdd(&P.st->lvl_iters[3], 1ull);
  int b = 0;
  while (b < 19 && (2ull << b) <= nl) b++;
  atomicAdd(&P.st->lvl_iters[4 + b], 1ull);
}

cudaError_t launch_walk_list_stats(const WalkParams &P, int gt, bool cont, int64_t n_targets, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(P.st->lvl_iters, 0, 24 * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
#define BH_GL_CASE(G)                                                                  \
  case G: {                                                                            \
    const unsigned grid = (unsigned)(((n_targets + G - 1) / G + 127) / 128);           \
    if (cont) k_glist_stats<G, true><<<grid, 128, 0, s>>>(P);                          \
    else k_glist_stats<G, false><<<grid, 128, 0, s>>>(P);                              \
  } break;
  switch (gt) {
    BH_GL_CASE(8)
    BH_GL_CASE(16)
    BH_GL_CASE(32)
    BH_GL_CASE(64)
    BH_GL_CASE(128)
    BH_GL_CASE(256)
    default: return cudaErrorInvalidValue;
  }
#undef BH_GL_CASE
  return cudaGetLastError();
}

}  // namespace bh
