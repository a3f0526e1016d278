// walk.cu -- K6 force walk (+ K7 fused leapfrog).
//
// PAPER.md:500-504 (§3): "The most computationally intensive part of the
// Barnes-Hut algorithm is the force computation stage."  PAPER.md:408-415:
// a remote cluster is treated as a single body only if D > r/theta.  Readings
// (DESIGN.md §3): r = cell side s_l = L 2^-l (L1), D = distance to the centre
// of mass (L2), strict s^2 < theta^2 D^2 (L3, L4), cells containing the target
// are always opened (L5), Plummer softening on every source (L6), G applied
// last (L7); "interactions" = accepted cells + particles j != i (L21).
//
// Per-particle semantics with warp-shared traversal.  Targets
// are taken in Morton order; a group of G lanes (G = 32: a warp) walks ONE
// stackless DFS over the record array: at record c every active lane evaluates
// its own MAC; lanes that accept c interact with it and become inactive until
// skip(c) (their subtree is done); the group descends (c + 1) if any active lane
// opens c, else jumps to skip(c).  Each lane therefore sees exactly its own
// Barnes-Hut frontier, in DFS order -- identical decisions to the oracle's
// recursive walk -- while the group's record loads are one broadcast address.
//
// MAC decisions are exact: the fp32 test uses the per-node thresholds T_acc /
// T_rej of com.cu; only when d2_32 falls between them is the oracle's fp64
// formula re-evaluated from the fp64 moments (counted in `fallbacks`).
//
// Interaction (fp32): r2 = d2 + eps^2, f = M rsqrt(r2)^3, a += f (dx, dy, dz):
// 18 flops + 1 MUFU.RSQ.  Partial sums are folded into fp64 every 64 interactions of
// the lane, so the result does not depend on the group size or the rank count.
//
// K7 (mode 1): v += a * kick (kick = dt/2 on the first step, dt after; reading
// L8), x += v dt, written in place to pos4 / vel4 of the particle's storage slot
// (the walk reads positions from the records, never from pos4).
#include <math.h>

#include "bh_internal.cuh"

namespace bh {

struct WalkParams {
  const float4 *__restrict__ rec_cm;
  const uint4 *__restrict__ rec_aux;
  const double4 *__restrict__ rec_mom;
  const uint32_t *__restrict__ nstart;
  const uint32_t *__restrict__ vals;
  const uint32_t *__restrict__ targets;
  const uint32_t *__restrict__ uid;
  DevStatus *st;
  uint32_t *icount;
  float4 *pos4;
  float4 *vel4;
  float *acc_out;  // mode 0: acc_out[3 uid[s]] (user_order) or acc_out[3 (s - own_lo)]
  int user_order;
  int64_t n_targets;
  int use_targets;
  int mode;
  float eps2, G, kick, dt;
  double theta2;
  uint32_t own_lo;
};

__device__ __noinline__ bool exact_accept(const double4 *__restrict__ rec_mom, uint32_t c, uint32_t level, float x,
                                          float y, float z, double L, double theta2) {
  // the oracle's fp64 test (DESIGN.md §3 L4), operation for operation
  double4 m = rec_mom[c];
  double cx = __ddiv_rn(m.y, m.x), cy = __ddiv_rn(m.z, m.x), cz = __ddiv_rn(m.w, m.x);
  double dx = __dsub_rn(cx, (double)x), dy = __dsub_rn(cy, (double)y), dz = __dsub_rn(cz, (double)z);
  double d2 = __dmul_rn(dx, dx);
  d2 = __dadd_rn(d2, __dmul_rn(dy, dy));
  d2 = __dadd_rn(d2, __dmul_rn(dz, dz));
  double s = ldexp(L, -(int)level);
  double s2 = __dmul_rn(s, s);
  return s2 < __dmul_rn(theta2, d2);
}

template <int G>
__global__ void __launch_bounds__(256) k_walk(const WalkParams P) {
  const uint32_t full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint32_t gmask = G == 32 ? full : (((1u << G) - 1u) << (lane & ~(G - 1)));
  if (P.st->err & ERR_NODE_OVERFLOW) return;
  const uint32_t Wn = P.st->n_records;
  const double Ld = (double)P.st->L;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool tvalid = t < P.n_targets;
  uint32_t p = 0, Li = 0, s = 0;
  float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tvalid) {
    p = P.use_targets ? P.targets[t] : (uint32_t)t;
    Li = P.nstart[p + 1] - 1u;
    me = P.rec_cm[Li];
    s = P.vals[p];
  }
  const bool gvalid = (__ballot_sync(full, tvalid) & gmask) != 0u;
  uint32_t c = gvalid ? 0u : Wn;
  uint32_t resume = 0, cnt = 0, fb = 0, nop = 0, nit = 0;
  int bad = 0;
  float ax = 0.f, ay = 0.f, az = 0.f;
  double dax = 0.0, day = 0.0, daz = 0.0;
  for (;;) {
    const bool live = c < Wn;
    if (G == 32) {
      if (!live) break;
    } else {
      if (!__any_sync(full, live)) break;
    }
    nit += live;
    const uint32_t cc = live ? c : 0u;
    const float4 cm = __ldg(&P.rec_cm[cc]);
    const uint4 au = __ldg(&P.rec_aux[cc]);
    const uint32_t skip = au.z;
    const float dx = cm.x - me.x, dy = cm.y - me.y, dz = cm.z - me.z;
    const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    const bool act = live && tvalid && c >= resume;
    const bool cont = (c <= Li) && (Li < skip);
    bool acc = act && !cont && d2 > __uint_as_float(au.x);
    const bool amb = act && !cont && !acc && !(d2 < __uint_as_float(au.y));
    if (amb) {
      acc = exact_accept(P.rec_mom, cc, au.w & META_LEVEL_MASK, me.x, me.y, me.z, Ld, P.theta2);
      fb++;
    }
    if (acc) {
      const float r2 = d2 + P.eps2;
      bad |= (r2 == 0.0f);
      const float inv = rsqrtf(r2);
      const float f = cm.w * (inv * inv) * inv;
      ax = fmaf(f, dx, ax);
      ay = fmaf(f, dy, ay);
      az = fmaf(f, dz, az);
      cnt++;
      resume = skip;
      if ((cnt & 63u) == 0u) {  // fold per lane: results independent of the group size
        dax += ax; day += ay; daz += az;
        ax = ay = az = 0.f;
      }
    }
    const bool opn = act && !acc;
    nop += opn;
    const uint32_t ob = __ballot_sync(full, opn);
    if (live) c = (ob & gmask) ? c + 1u : skip;
  }
  dax += ax; day += ay; daz += az;
  // warp reductions of the counters
  unsigned long long wc = cnt, wf = fb, wo = nop, wi = nit;
  for (int o = 16; o; o >>= 1) {
    wc += __shfl_xor_sync(full, wc, o);
    wf += __shfl_xor_sync(full, wf, o);
    wo += __shfl_xor_sync(full, wo, o);
    wi += __shfl_xor_sync(full, wi, o);
  }
  const int wbad = __any_sync(full, bad);
  if (lane == 0) {
    if (wc) { atomicAdd(&P.st->interactions, wc); atomicAdd(&P.st->interactions_cum, wc); }
    if (wf) atomicAdd(&P.st->fallbacks, wf);
    if (wo) { atomicAdd(&P.st->opens, wo); atomicAdd(&P.st->opens_cum, wo); }
    if (wi) atomicAdd(&P.st->iters, wi);
    if (wbad) atomicOr(&P.st->err, ERR_NONFINITE_FORCE);
  }
  if (!tvalid) return;
  const float gx = P.G * (float)dax, gy = P.G * (float)day, gz = P.G * (float)daz;
  P.icount[s] = cnt;
  const uint32_t o = s - P.own_lo;
  if (P.mode == 0) {
    if (P.acc_out) {
      const size_t k = P.user_order ? (size_t)P.uid[s] : (size_t)o;
      P.acc_out[3 * k + 0] = gx;
      P.acc_out[3 * k + 1] = gy;
      P.acc_out[3 * k + 2] = gz;
    }
  } else {
    float4 v = P.vel4[o];
    v.x = fmaf(gx, P.kick, v.x);
    v.y = fmaf(gy, P.kick, v.y);
    v.z = fmaf(gz, P.kick, v.z);
    P.vel4[o] = v;
    P.pos4[s] = make_float4(fmaf(v.x, P.dt, me.x), fmaf(v.y, P.dt, me.y), fmaf(v.z, P.dt, me.z), me.w);
  }
}

cudaError_t launch_walk(const Workspace &W, const WalkArgs &a, cudaStream_t s) {
  if (a.n_targets <= 0) return cudaSuccess;
  WalkParams P;
  P.rec_cm = W.rec_cm;
  P.rec_aux = W.rec_aux;
  P.rec_mom = W.rec_mom;
  P.nstart = W.nstart;
  P.vals = W.vals[a.buf];
  P.targets = W.targets;
  P.uid = W.uid;
  P.st = W.status;
  P.icount = W.icount;
  P.pos4 = W.pos4;
  P.vel4 = W.vel4;
  P.acc_out = a.acc_out;
  P.user_order = a.user_order;
  P.n_targets = a.n_targets;
  P.use_targets = a.use_targets;
  P.mode = a.mode;
  P.eps2 = a.eps2;
  P.G = a.G;
  P.kick = a.kick;
  P.dt = a.dt;
  P.theta2 = a.theta2;
  P.own_lo = a.own_lo;
  unsigned grid = (unsigned)((a.n_targets + 255) / 256);
  switch (a.group) {
    case 1: k_walk<1><<<grid, 256, 0, s>>>(P); break;
    case 2: k_walk<2><<<grid, 256, 0, s>>>(P); break;
    case 4: k_walk<4><<<grid, 256, 0, s>>>(P); break;
    case 8: k_walk<8><<<grid, 256, 0, s>>>(P); break;
    case 16: k_walk<16><<<grid, 256, 0, s>>>(P); break;
    default: k_walk<32><<<grid, 256, 0, s>>>(P); break;
  }
  return cudaGetLastError();
}

}  // namespace bh
