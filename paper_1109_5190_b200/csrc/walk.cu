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
// MAC decisions are exact.  The fast kernel decides with the fp32 thresholds
// T_acc / T_rej of com.cu (d2_32 > T_acc: accept for sure; d2_32 < T_rej: open
// for sure).  A lane whose d2_32 falls between them (~1e-6 of the tests) drops
// out of the fast walk at that record and is queued with its partial sums;
// k_walk_resume then continues each such target's DFS from that record alone,
// with the oracle's fp64 test on the ambiguous nodes.  The fast loop thus
// carries no fp64 code and no divergent branch.
//
// Interaction (fp32): r2 = d2 + eps^2, f = M rsqrt(r2)^3, a += f (dx, dy, dz):
// 18 flops + 1 MUFU.RSQ, summed sequentially in fp32 in the lane's own DFS
// order (so the result does not depend on the group size or the rank count).
// Measured max per-particle error vs the fp64 oracle: <= 2.5e-5 on cfg1-cfg4
// (DESIGN.md §6); -DBH_FOLD64 folds the fp32 partials into fp64 every 64
// interactions (max error <= 1.8e-5 -> 2.7e-6 on cfg2, 17% slower walk).
//
// K7 (mode 1): v += a * kick (kick = dt/2 on the first step, dt after; reading
// L8), x += v dt, written in place to pos4 / vel4 of the particle's storage slot
// (the walk reads positions from the records, never from pos4).
#include <math.h>
#include <stdlib.h>

#include "bh_internal.cuh"

namespace bh {

struct WalkParams {
  const Rec *__restrict__ rec;
  const float4 *__restrict__ qrec;  // multipole = 2: -Q (fp32) per record, 2 float4 (else null)
  int quad;
  const double4 *__restrict__ rec_mom;
  const uint32_t *__restrict__ nstart;
  const uint32_t *__restrict__ vals;
  const uint32_t *__restrict__ targets;
  const uint32_t *__restrict__ uid;
  DevStatus *st;
  uint32_t *icount;
  uint32_t *redo;
  ResumeState *resume;
  int64_t cap_resume;
  int resume_stack;
  int need_cont;
  float4 *pos4;
  float4 *vel4;
  float *acc_out;  // mode 0: acc_out[3 uid[s]] (user_order) or acc_out[3 (s - own_lo)]
  uint32_t *gcost;  // k_walk2: per storage id, the last-walk trips of its group (or null)
  int user_order;
  int64_t n_targets;
  int use_targets;
  int mode;
  float eps2, G, kick, dt;
  double theta2;
  uint32_t own_lo;
  int num_sms;
};

__device__ __forceinline__ float rsqrt_fast(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// multipole = 2 (reading L25): the quadrupole field of an accepted cell,
//   a += -(Q dr) / r_e^5 + (5/2) (dr^T Q dr) dr / r_e^7,   dr = (dx, dy, dz),
// with nq = -Q (the records hold -Q): q = nq dr, s = dr^T q = -(dr^T Q dr),
// g1 = inv^5, g2 = (-2.5 s) inv^7:  a += g1 q + g2 dr.  Every walk kernel uses
// this operation sequence (k_walk2 in packed pairs), so they agree bitwise.
struct QuadRec {
  float xx, yy, zz, xy, xz, yz;
};
__device__ __forceinline__ QuadRec load_quad(const float4 *__restrict__ qrec, uint32_t c) {
  const float4 a = qrec[2 * (size_t)c], b = qrec[2 * (size_t)c + 1];
  QuadRec q;
  q.xx = a.x; q.yy = a.y; q.zz = a.z; q.xy = a.w; q.xz = b.x; q.yz = b.y;
  return q;
}
__device__ __forceinline__ void quad_term(const QuadRec &Q, float dx, float dy, float dz, float inv, bool acc,
                                          float &ax, float &ay, float &az) {
  const float qx = __fmaf_rn(Q.xz, dz, __fmaf_rn(Q.xy, dy, __fmul_rn(Q.xx, dx)));
  const float qy = __fmaf_rn(Q.yz, dz, __fmaf_rn(Q.yy, dy, __fmul_rn(Q.xy, dx)));
  const float qz = __fmaf_rn(Q.zz, dz, __fmaf_rn(Q.yz, dy, __fmul_rn(Q.xz, dx)));
  const float sq = __fmaf_rn(qz, dz, __fmaf_rn(qy, dy, __fmul_rn(qx, dx)));
  const float inv2 = __fmul_rn(inv, inv);
  const float inv5 = __fmul_rn(__fmul_rn(inv2, inv2), inv);
  const float inv7 = __fmul_rn(inv5, inv2);
  const float g1 = acc ? inv5 : 0.0f;  // branch-free, like the monopole's f
  const float g2 = acc ? __fmul_rn(__fmul_rn(-2.5f, sq), inv7) : 0.0f;
  ax = __fmaf_rn(g2, dx, __fmaf_rn(g1, qx, ax));
  ay = __fmaf_rn(g2, dy, __fmaf_rn(g1, qy, ay));
  az = __fmaf_rn(g2, dz, __fmaf_rn(g1, qz, az));
}

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

struct Target {
  uint32_t p, Li, s;
  float4 me;
};

__device__ __forceinline__ Target load_target(const WalkParams &P, int64_t t) {
  Target T;
  T.p = P.use_targets ? P.targets[t] : (uint32_t)t;
  T.Li = P.nstart[T.p + 1] - 1u;  // the particle's own record
  T.me = P.rec[T.Li].cm;
  T.s = P.vals[T.p];
  return T;
}

// outputs of one target: forces (mode 0) or the fused leapfrog (mode 1)
__device__ __forceinline__ void finish(const WalkParams &P, const Target &T, double dax, double day, double daz,
                                       uint32_t cnt) {
  if (!(isfinite(dax) && isfinite(day) && isfinite(daz))) atomicOr(&P.st->err, ERR_NONFINITE_FORCE);
  const float gx = P.G * (float)dax, gy = P.G * (float)day, gz = P.G * (float)daz;
  P.icount[T.s] = cnt;
  const uint32_t o = T.s - P.own_lo;
  if (P.mode == 0) {
    if (P.acc_out) {
      const size_t k = P.user_order ? (size_t)P.uid[T.s] : (size_t)o;
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
    P.pos4[T.s] = make_float4(fmaf(v.x, P.dt, T.me.x), fmaf(v.y, P.dt, T.me.y), fmaf(v.z, P.dt, T.me.z), T.me.w);
  }
}

// A target whose fp32 MAC test was inconclusive at record cdrop (its resume
// word is BH_DROP | cdrop) is queued with its fp32 partial sums and count over
// the DFS prefix before cdrop; k_walk_resume continues the same DFS from
// cdrop with the oracle's exact test.  `own` = 1 if the count includes the
// target's own record (the CONT = false kernels accept it with a zero
// contribution; the resume kernel opens it, as the oracle does).
__device__ __forceinline__ void push_resume(const WalkParams &P, int64_t t, uint32_t res, float ax, float ay, float az,
                                            uint32_t cnt, uint32_t own) {
  const unsigned long long k = atomicAdd(&P.st->n_redo, 1ull);
  P.redo[k] = (uint32_t)t;
  if ((int64_t)k < P.cap_resume) {
    ResumeState r;
    r.ax = ax;
    r.ay = ay;
    r.az = az;
    r.cnt = cnt - own;
    r.cdrop = res & ~BH_DROP;
    r.pad[0] = r.pad[1] = r.pad[2] = 0u;
    P.resume[k] = r;
  }
}

template <int G, bool STATS>
__global__ void __launch_bounds__(256) k_walk(const WalkParams P) {
  const uint32_t full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint32_t gmask = G == 32 ? full : (((1u << G) - 1u) << (lane & ~(G - 1)));
  if (P.st->err & ERR_NODE_OVERFLOW) return;
  const uint32_t Wn = P.st->n_records;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool tvalid = t < P.n_targets;
  Target T;
  if (tvalid) T = load_target(P, t);
  else { T.p = 0; T.Li = 0; T.s = 0; T.me = make_float4(0.f, 0.f, 0.f, 0.f); }
  const uint32_t Li = T.Li;
  const float mx = T.me.x, my = T.me.y, mz = T.me.z;
  const bool gvalid = (__ballot_sync(full, tvalid) & gmask) != 0u;
  const float eps2 = P.eps2;
  const Rec *__restrict__ rec = P.rec;
  asm volatile("" : "+l"(rec));  // keep the base in a register (no per-iteration constant reload)
  uint32_t c = gvalid ? 0u : Wn;
  // a lane is active at record c iff c >= resume; an invalid (or dropped-out)
  // lane has resume past every record
  uint32_t resume = tvalid ? 0u : 0xffffffffu;
  uint32_t cnt = 0, nop = 0, nit = 0;
  float ax = 0.f, ay = 0.f, az = 0.f;
  double dax = 0.0, day = 0.0, daz = 0.0;
  bool live = c < Wn;
  __shared__ unsigned long long s_lv[3][24];
  if (STATS) {
    for (int i = threadIdx.x; i < 72; i += blockDim.x) (&s_lv[0][0])[i] = 0ull;
    __syncthreads();
  }
  // outer loop: the fp64 fold runs on a uniform exit of the inner loop
  while (G == 32 ? live : __any_sync(full, live)) {
    bool fold;
    for (;;) {
      if (STATS) nit++;
      const uint32_t cc = (G == 32) ? c : (live ? c : 0u);
      const float4 cm = __ldg(&rec[cc].cm);
      const uint4 au = __ldg(&rec[cc].aux);
      const uint32_t skip = au.z;
      const float dx = cm.x - mx, dy = cm.y - my, dz = cm.z - mz;
      const float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      // act: past the subtree of the last accepted node; cont: c <= Li < skip
      const bool act = (G == 32 ? true : live) & (cc >= resume);
      const bool ok = act & !((cc <= Li) & (skip > Li));
      const bool acc = ok & (d2 > __uint_as_float(au.x));
      const bool amb = ok & !acc & (d2 >= __uint_as_float(au.y));
      const bool opn = act & !acc & !amb;
      if (STATS) {
        nop += opn;
        const uint32_t lv = au.w & META_LEVEL_MASK;
        const uint32_t na = __popc(__ballot_sync(full, act) & gmask), ni = __popc(__ballot_sync(full, acc) & gmask);
        if ((lane & (G - 1)) == 0 && (G == 32 || live)) {
          atomicAdd(&s_lv[0][lv], (unsigned long long)G);
          atomicAdd(&s_lv[1][lv], (unsigned long long)na);
          atomicAdd(&s_lv[2][lv], (unsigned long long)ni);
        }
      }
      // interaction, branch-free: f = 0 for lanes that do not accept c
      const float inv = rsqrt_fast(d2 + eps2);
      float f = cm.w * (inv * inv) * inv;
      f = acc ? f : 0.0f;
      ax = fmaf(f, dx, ax);
      ay = fmaf(f, dy, ay);
      az = fmaf(f, dz, az);
      if (P.quad) quad_term(load_quad(P.qrec, cc), dx, dy, dz, inv, acc, ax, ay, az);
      asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q add.u32 %0, %0, 1;\n\t}" : "+r"(cnt) : "r"((uint32_t)acc));
      resume = acc ? skip : (amb ? (BH_DROP | cc) : resume);
      uint32_t nxt;
      if (G == 32) {
        nxt = __any_sync(full, opn) ? cc + 1u : skip;
        c = nxt;
      } else {
        nxt = (__ballot_sync(full, opn) & gmask) ? cc + 1u : skip;
        c = live ? nxt : c;
      }
      live = c < Wn;
#ifdef BH_FOLD64
      fold = acc & ((cnt & 63u) == 0u);
      if (__any_sync(full, fold)) break;
#else
      fold = false;
#endif
      if (G == 32 ? !live : !__any_sync(full, live)) break;
    }
    if (fold) {
      dax += ax; day += ay; daz += az;
      ax = ay = az = 0.f;
    }
  }
  dax += ax; day += ay; daz += az;
  // warp reductions of the counters
  // a lane that met an inconclusive MAC test dropped out with resume = BH_DROP | c
  const bool redo = tvalid && resume >= BH_DROP;
  unsigned long long wc = redo ? 0u : cnt, wo = nop, wi = nit;
  for (int o = 16; o; o >>= 1) {
    wc += __shfl_xor_sync(full, wc, o);
    if (STATS) {
      wo += __shfl_xor_sync(full, wo, o);
      wi += __shfl_xor_sync(full, wi, o);
    }
  }
  if (STATS) {
    __syncthreads();
    for (int i = threadIdx.x; i < 72; i += blockDim.x) {
      unsigned long long v = (&s_lv[0][0])[i];
      if (v) atomicAdd(&P.st->lvl_iters[0] + i, v);
    }
  }
  if (lane == 0) {
    if (wc) { atomicAdd(&P.st->interactions, wc); atomicAdd(&P.st->interactions_cum, wc); }
    if (STATS && wo) { atomicAdd(&P.st->opens, wo); atomicAdd(&P.st->opens_cum, wo); }
    if (STATS && wi) atomicAdd(&P.st->iters, wi);
  }
  if (!tvalid) return;
  if (redo) {  // continued by k_walk_resume
    push_resume(P, t, resume, (float)dax, (float)day, (float)daz, cnt, 0u);
    return;
  }
  finish(P, T, dax, day, daz, cnt);
}

// ---------------------------------------------------------------- k_walk2
// The production walk: the same per-lane semantics and the same fp32 operation
// sequence per target as k_walk (bitwise-identical results), but every lane
// carries TWO targets and does their arithmetic with Blackwell's packed fp32
// instructions (FADD2 / FMUL2 / FFMA2: one issue slot, two fp32 results; the
// node's fields enter as broadcast scalar operands).  The record loads, the
// traversal control and the vote are shared by the pair, so the issue slots per
// target-visit drop by ~1/3.  A group of GL lanes (2 GL targets, Morton-
// consecutive) shares one traversal.
struct F2 {
  unsigned long long v;
};
__device__ __forceinline__ F2 pk2(float lo, float hi) {
  F2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(F2 a, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.v));
}
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
  F2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 add2(F2 a, F2 b) {
  F2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
  F2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}
__device__ __forceinline__ void fma2_acc(F2 &acc, F2 a, F2 b) {  // acc = a * b + acc, in place
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc.v) : "l"(a.v), "l"(b.v));
}

__device__ __forceinline__ void ld_rec(const Rec *p, float4 &cm, uint4 &au) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(cm.x), "=f"(cm.y), "=f"(cm.z), "=f"(cm.w), "=r"(au.x), "=r"(au.y), "=r"(au.z), "=r"(au.w)
               : "l"(p));
}

// One target's MAC decision at record cc, as bit masks (few live predicates):
//   act = cc >= res (and, with CONT, the record does not contain the target)
//   acc = act & d2 > T_acc      -> interact (f kept), cnt += 1, res = skip
//   amb = act & !acc & d2 >= T_rej -> inconclusive: res = BH_DROP | cc (the
//                                   target drops out; k_walk_resume continues it)
//   opn |= act & d2 < T_rej     -> the lane descends
// Identical decisions to k_walk / k_walk2.
__device__ __forceinline__ void mac_pair(uint32_t cc, float d2A, float d2B, float tacc, float trej, uint32_t skip,
                                         uint32_t &resA, uint32_t &resB, uint32_t &cntA, uint32_t &cntB,
                                         uint32_t &opn, float &fA, float &fB) {
  const uint32_t drop = BH_DROP | cc;
  asm("{\n\t.reg .pred pa, pc, pq, pb, pd, pr, po;\n\t"
      "setp.ge.u32 pa, %9, %0;\n\t"                 // act A
      "setp.gt.and.f32 pc, %10, %12, pa;\n\t"       // acc A
      "setp.ge.and.f32 pq, %10, %13, pa;\n\t"       // acc-or-amb A
      "setp.ge.u32 pb, %9, %1;\n\t"                 // act B
      "setp.gt.and.f32 pd, %11, %12, pb;\n\t"       // acc B
      "setp.ge.and.f32 pr, %11, %13, pb;\n\t"       // acc-or-amb B
      "@pc add.u32 %2, %2, 1;\n\t"
      "@pd add.u32 %3, %3, 1;\n\t"
      "@pq selp.b32 %0, %14, %15, pc;\n\t"   // acc: skip; amb: BH_DROP | cc (dropped out)
      "@pr selp.b32 %1, %14, %15, pd;\n\t"
      "@!pc mov.b32 %5, 0f00000000;\n\t"
      "@!pd mov.b32 %6, 0f00000000;\n\t"
      "not.pred pq, pq;\n\t"
      "not.pred pr, pr;\n\t"
      "and.pred pa, pa, pq;\n\t"
      "and.pred pb, pb, pr;\n\t"
      "or.pred po, pa, pb;\n\t"
      "@po mov.b32 %4, 1;\n\t}"
      : "+r"(resA), "+r"(resB), "+r"(cntA), "+r"(cntB), "+r"(opn), "+f"(fA), "+f"(fB)
      : "r"(cc), "r"(cc), "r"(cc), "f"(d2A), "f"(d2B), "f"(tacc), "f"(trej), "r"(skip), "r"(drop));
}

// mac_pair that also zeroes the quadrupole factors (g1, g2) of targets that do
// not accept the record
__device__ __forceinline__ void mac_pair_q(uint32_t cc, float d2A, float d2B, float tacc, float trej, uint32_t skip,
                                           uint32_t &resA, uint32_t &resB, uint32_t &cntA, uint32_t &cntB,
                                           uint32_t &opn, float &fA, float &fB, float &g1A, float &g1B, float &g2A,
                                           float &g2B) {
  const uint32_t drop = BH_DROP | cc;
  asm("{\n\t.reg .pred pa, pc, pq, pb, pd, pr, po;\n\t"
      "setp.ge.u32 pa, %13, %0;\n\t"
      "setp.gt.and.f32 pc, %14, %16, pa;\n\t"
      "setp.ge.and.f32 pq, %14, %17, pa;\n\t"
      "setp.ge.u32 pb, %13, %1;\n\t"
      "setp.gt.and.f32 pd, %15, %16, pb;\n\t"
      "setp.ge.and.f32 pr, %15, %17, pb;\n\t"
      "@pc add.u32 %2, %2, 1;\n\t"
      "@pd add.u32 %3, %3, 1;\n\t"
      "@pq selp.b32 %0, %18, %19, pc;\n\t"
      "@pr selp.b32 %1, %18, %19, pd;\n\t"
      "@!pc mov.b32 %5, 0f00000000;\n\t"
      "@!pd mov.b32 %6, 0f00000000;\n\t"
      "@!pc mov.b32 %7, 0f00000000;\n\t"
      "@!pd mov.b32 %8, 0f00000000;\n\t"
      "@!pc mov.b32 %9, 0f00000000;\n\t"
      "@!pd mov.b32 %10, 0f00000000;\n\t"
      "not.pred pq, pq;\n\t"
      "not.pred pr, pr;\n\t"
      "and.pred pa, pa, pq;\n\t"
      "and.pred pb, pb, pr;\n\t"
      "or.pred po, pa, pb;\n\t"
      "@po mov.b32 %4, 1;\n\t}"
      : "+r"(resA), "+r"(resB), "+r"(cntA), "+r"(cntB), "+r"(opn), "+f"(fA), "+f"(fB), "+f"(g1A), "+f"(g1B),
        "+f"(g2A), "+f"(g2B)
      : "r"(cc), "r"(cc), "r"(cc), "f"(d2A), "f"(d2B), "f"(tacc), "f"(trej), "r"(skip), "r"(drop));
}

#ifndef BH_WALK2_BLOCK
#define BH_WALK2_BLOCK 128
#endif
#ifndef BH_WALK2_UNROLL
#define BH_WALK2_UNROLL 2
#endif
#ifndef BH_WALK2_MINB
#define BH_WALK2_MINB 5
#endif
// NP pairs of targets per lane (2 NP targets), GL lanes per group: a group of
// 2 NP GL Morton-consecutive targets shares one traversal.
template <int GL, int NP, bool CONT, bool QUAD>
__global__ void __launch_bounds__(BH_WALK2_BLOCK, (NP == 1 && !QUAD ? BH_WALK2_MINB : 4) * 256 / BH_WALK2_BLOCK) k_walk2(const WalkParams P) {
  constexpr int TPL = 2 * NP;  // targets per lane
  const uint32_t full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const uint32_t gmask = GL == 32 ? full : (((1u << GL) - 1u) << (lane & ~(GL - 1)));
  if (P.st->err & ERR_NODE_OVERFLOW) return;
  const uint32_t Wn = P.st->n_records;
  const uint32_t chunk = blockIdx.x;
  // Group order.  The block's 256 / GL groups are dealt to its warps in
  // descending order of their predicted cost (union-walk trips in the last
  // walk, kept per particle in gcost):
  // a warp runs until its slowest group is done, so warps of similar groups
  // idle less (the groups themselves -- which targets walk together -- do not
  // change, hence neither do the results).  Without costs: Morton order.
  constexpr int GPB = BH_WALK2_BLOCK / GL;  // groups per block
  const int gi = lane / GL, gl = lane % GL;
  int lg = (threadIdx.x >> 5) * (32 / GL) + gi;  // local group of this lane
  if (P.gcost) {
    __shared__ uint32_t s_cost[GPB], s_perm[GPB];
    const int64_t g0 = (int64_t)chunk * GPB;
    const int64_t ngroups = (P.n_targets + GL * TPL - 1) / (GL * TPL);
    if (threadIdx.x < GPB) {
      // a group's predicted cost: the last-walk cost recorded on its first and
      // last targets (costs travel with the particles, groups are re-formed
      // from the current Morton order every step)
      uint32_t cst = 0u;
      const int64_t g = g0 + threadIdx.x;
      if (g < ngroups) {
        const int64_t t0 = g * (GL * TPL);
        const int64_t t1 = min(t0 + GL * TPL, P.n_targets) - 1;
        const uint32_t p0 = P.use_targets ? P.targets[t0] : (uint32_t)t0;
        const uint32_t p1 = P.use_targets ? P.targets[t1] : (uint32_t)t1;
        cst = max(P.gcost[P.vals[p0]], P.gcost[P.vals[p1]]);
      }
      s_cost[threadIdx.x] = cst;
    }
    __syncthreads();
    if (threadIdx.x < GPB) {
      const uint32_t ci = s_cost[threadIdx.x];
      int r = 0;
      for (int j = 0; j < GPB; j++) {
        const uint32_t cj = s_cost[j];
        r += (cj > ci) | ((cj == ci) & (j < (int)threadIdx.x));
      }
      s_perm[r] = threadIdx.x;
    }
    __syncthreads();
    lg = (int)s_perm[lg];
  }
  const int64_t gidx = (int64_t)chunk * GPB + lg;  // global group index
  const int64_t tbase = gidx * (GL * TPL) + gl;
  Target T[TPL];
  bool v[TPL];
  bool anyv = false;
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    const int64_t t = tbase + (int64_t)k * GL;
    v[k] = t < P.n_targets;
    anyv |= v[k];
    if (v[k]) T[k] = load_target(P, t);
    else { T[k].p = 0; T[k].Li = 0; T[k].s = 0; T[k].me = make_float4(0.f, 0.f, 0.f, 0.f); }
  }
  uint32_t Li[TPL], res[TPL], cnt[TPL];
  float ax[TPL], ay[TPL], az[TPL];
  F2 X[NP], Y[NP], Z[NP];
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    Li[k] = T[k].Li;
    res[k] = v[k] ? 0u : 0xffffffffu;
    cnt[k] = 0;
    ax[k] = ay[k] = az[k] = 0.f;
  }
#pragma unroll
  for (int j = 0; j < NP; j++) {
    X[j] = pk2(T[2 * j].me.x, T[2 * j + 1].me.x);
    Y[j] = pk2(T[2 * j].me.y, T[2 * j + 1].me.y);
    Z[j] = pk2(T[2 * j].me.z, T[2 * j + 1].me.z);
  }
  const F2 E2 = pk2(P.eps2, P.eps2);
  const bool gvalid = (__ballot_sync(full, anyv) & gmask) != 0u;
  const Rec *__restrict__ rec = P.rec;
  asm volatile("" : "+l"(rec));  // base in a register (no per-iteration constant reload)
  uint32_t gmask2 = gmask;
  asm volatile("" : "+r"(gmask2));  // a plain register: the group test is one LOP3
  uint32_t c = gvalid ? 0u : Wn;
  uint32_t git = 0;  // union-walk trips (2 visits) of this lane's group (its cost)
  // a finished group parks on the sentinel record Wn (T_acc = T_rej = +inf,
  // skip = Wn: nothing is accepted or queued there) until the warp is done
  // two visits per trip: the exit vote and the cost counter run once per trip
  // (a parked group stays on the sentinel, so the extra visit is harmless)
  if (__any_sync(full, c < Wn)) for (;;) {
#pragma unroll
   for (int u = 0; u < BH_WALK2_UNROLL; u++) {
    const uint32_t cc = c;
    float4 cm;
    uint4 au;
    ld_rec(rec + cc, cm, au);
    const uint32_t skip = au.z;
    const float tacc = __uint_as_float(au.x), trej = __uint_as_float(au.y);
    uint32_t opn = 0u;
#pragma unroll
    for (int j = 0; j < NP; j++) {
      const int a = 2 * j, b = 2 * j + 1;
      const F2 DX = sub2(pk2(cm.x, cm.x), X[j]), DY = sub2(pk2(cm.y, cm.y), Y[j]),
               DZ = sub2(pk2(cm.z, cm.z), Z[j]);
      const F2 D2 = fma2(DZ, DZ, fma2(DY, DY, mul2(DX, DX)));
      float d2A, d2B;
      up2(D2, d2A, d2B);
      // interaction for both targets of the pair, branch-free (f zeroed below
      // for a target that does not accept the record)
      float r2A, r2B;
      up2(add2(D2, E2), r2A, r2B);
      const F2 INV = pk2(rsqrt_fast(r2A), rsqrt_fast(r2B));
      float fA, fB;
      const F2 INV2 = mul2(INV, INV);
      up2(mul2(mul2(pk2(cm.w, cm.w), INV2), INV), fA, fB);
      // multipole = 2: the record's -Q (broadcast) and the quadrupole factors
      // (quad_term's operation sequence, in pairs)
      F2 QX, QY, QZ;
      float g1A = 0.f, g1B = 0.f, g2A = 0.f, g2B = 0.f;
      if (QUAD) {
        const float4 qa = __ldg(&P.qrec[2 * (size_t)cc]), qb = __ldg(&P.qrec[2 * (size_t)cc + 1]);
        // qa = (xx, yy, zz, xy), qb = (xz, yz, -, -)
        QX = fma2(pk2(qb.x, qb.x), DZ, fma2(pk2(qa.w, qa.w), DY, mul2(pk2(qa.x, qa.x), DX)));
        QY = fma2(pk2(qb.y, qb.y), DZ, fma2(pk2(qa.y, qa.y), DY, mul2(pk2(qa.w, qa.w), DX)));
        QZ = fma2(pk2(qa.z, qa.z), DZ, fma2(pk2(qb.y, qb.y), DY, mul2(pk2(qb.x, qb.x), DX)));
        const F2 SQ = fma2(QZ, DZ, fma2(QY, DY, mul2(QX, DX)));
        const F2 INV5 = mul2(mul2(INV2, INV2), INV);
        const F2 INV7 = mul2(INV5, INV2);
        up2(INV5, g1A, g1B);
        up2(mul2(mul2(pk2(-2.5f, -2.5f), SQ), INV7), g2A, g2B);
      }
      // per-target MAC (identical decisions to k_walk); an inconclusive fp32
      // test drops the target out (resume = BH_DROP | c): k_walk_resume continues it
      // (a record containing the target is opened, never accepted: NaN distance)
      float qA = d2A, qB = d2B;
      if (CONT) {
        const bool cA = (cc <= Li[a]) & (skip > Li[a]), cB = (cc <= Li[b]) & (skip > Li[b]);
        const float qnan = __int_as_float(0x7fffffff);
        qA = cA ? qnan : d2A;
        qB = cB ? qnan : d2B;
      }
      if (QUAD) {
        mac_pair_q(cc, qA, qB, tacc, trej, skip, res[a], res[b], cnt[a], cnt[b], opn, fA, fB, g1A, g1B, g2A, g2B);
      } else {
        mac_pair(cc, qA, qB, tacc, trej, skip, res[a], res[b], cnt[a], cnt[b], opn, fA, fB);
      }
      const F2 FF = pk2(fA, fB);
      // packed accumulate on (a, b) register pairs (this form avoids ptxas moves)
      asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
          : "+f"(ax[a]), "+f"(ax[b]) : "l"(FF.v), "l"(DX.v));
      asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
          : "+f"(ay[a]), "+f"(ay[b]) : "l"(FF.v), "l"(DY.v));
      asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
          : "+f"(az[a]), "+f"(az[b]) : "l"(FF.v), "l"(DZ.v));
      if (QUAD) {
        const F2 G1 = pk2(g1A, g1B), G2 = pk2(g2A, g2B);
        F2 AX = pk2(ax[a], ax[b]), AY = pk2(ay[a], ay[b]), AZ = pk2(az[a], az[b]);
        AX = fma2(G2, DX, fma2(G1, QX, AX));
        AY = fma2(G2, DY, fma2(G1, QY, AY));
        AZ = fma2(G2, DZ, fma2(G1, QZ, AZ));
        up2(AX, ax[a], ax[b]);
        up2(AY, ay[a], ay[b]);
        up2(AZ, az[a], az[b]);
      }
    }
    if (GL == 32) {
      c = min(__any_sync(full, opn != 0u) ? cc + 1u : skip, Wn);
    } else {
      const uint32_t nxt = (__ballot_sync(full, opn != 0u) & gmask2) ? cc + 1u : skip;
      c = min(nxt, Wn);
    }
   }
    const bool live = c < Wn;
    git += live ? 1u : 0u;
    if (!__any_sync(full, live)) break;
  }
  if (P.gcost) {
#pragma unroll
    for (int k = 0; k < TPL; k++)
      if (v[k]) P.gcost[T[k].s] = git;  // this walk's cost of the target's group
  }
  unsigned long long wc = 0;
  bool redo[TPL];
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    redo[k] = v[k] && res[k] >= BH_DROP;
    if (!CONT && !redo[k]) cnt[k] -= v[k] ? 1u : 0u;  // own record: "accepted", zero contribution
    wc += redo[k] ? 0u : cnt[k];
  }
  for (int o = 16; o; o >>= 1) wc += __shfl_xor_sync(full, wc, o);
  if (lane == 0 && wc) {
    atomicAdd(&P.st->interactions, wc);
    atomicAdd(&P.st->interactions_cum, wc);
  }
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    if (!v[k]) continue;
    if (redo[k])
      push_resume(P, tbase + (int64_t)k * GL, res[k], ax[k], ay[k], az[k], cnt[k],
                  (!CONT && Li[k] < (res[k] & ~BH_DROP)) ? 1u : 0u);
    else finish(P, T[k], (double)ax[k], (double)ay[k], (double)az[k], cnt[k]);
  }
}

// ---------------------------------------------------------------- k_walk_lane
// Variant family (walk_group 80..85, 90..95): groups of GL lanes x TPL = 2 NP
// targets with a leaner MAC (mac_pair: predicates in one asm block, 7 ALU ops
// per target instead of 9-10) and one LDG.256 per record visit; the per-target
// semantics and the fp32 operation sequence are exactly those of k_walk /
// k_walk2 (bitwise-identical results).  80..85 are persistent (a lane group
// that finishes takes the next group from per-SM Morton segments, so no group
// idles behind a slower one in its warp); 90..95 give every group slot one
// group, like k_walk2.
// Measured on cfg4 (profiles/r1_walk_variants.md): none beats
// k_walk2<4,1> (49.3 ms).  The loop is bound by L1 register writeback (32 B per
// lane per visit: 64-75 % of the LSU writeback peak) and by load latency,
// not by issue: cutting instructions by 8-12 % (83, 93) gains nothing, 4
// targets per lane (80, 82, 92) halves the writeback but needs 80 registers
// (24 warps/SM) and loses L1 hits (34-45 % with persistent scheduling, whose
// warps are at unrelated depths of their walks, vs 86 % for k_walk2's
// phase-aligned blocks).  Kept as measured alternatives.
template <int GL, int NP, bool CONT, bool PERSIST>
__global__ void __launch_bounds__(256, (NP == 1 || !PERSIST) ? 4 : 3) k_walk_lane(const WalkParams P) {
  constexpr int TPL = 2 * NP;       // targets per lane
  constexpr int GT = GL * TPL;      // targets per group
  const uint32_t full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int gl = lane % GL;         // lane within the group
  const int glead = lane & ~(GL - 1);
  const uint32_t gmask = GL == 32 ? full : (((1u << GL) - 1u) << glead);
  if (P.st->err & ERR_NODE_OVERFLOW) return;
  const uint32_t Wn = P.st->n_records;
  const int64_t ngroups = (P.n_targets + GT - 1) / GT;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  uint32_t Li[TPL], res[TPL], cnt[TPL];
  float ax[TPL], ay[TPL], az[TPL];
  F2 X[NP], Y[NP], Z[NP];
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    Li[k] = 0;
    res[k] = 0xffffffffu;
    cnt[k] = 0;
    ax[k] = ay[k] = az[k] = 0.f;
  }
#pragma unroll
  for (int j = 0; j < NP; j++) X[j] = Y[j] = Z[j] = pk2(0.f, 0.f);
  const F2 E2 = pk2(P.eps2, P.eps2);
  const Rec *__restrict__ rec = P.rec;
  asm volatile("" : "+l"(rec));  // base in a register (no per-iteration constant reload)
  uint32_t gm = gmask;
  asm volatile("" : "+r"(gm));      // a plain register: the group test is one LOP3
  int64_t g = -1;                   // current group (-1: none yet)
  bool parked = false;              // no groups left for this lane's group
  const int nseg = P.num_sms < 256 ? P.num_sms : 256;
  int seg, hops = 0;                // ticket segment (warp-uniform), segments exhausted
  bool first_done = false;
  asm("mov.u32 %0, %%smid;" : "=r"(seg));
  seg %= nseg;
  uint32_t c = Wn;                  // cursor (group-uniform); Wn = the sentinel record
  unsigned long long wc = 0;
  for (;;) {
    const bool need = (c >= Wn) & !parked;   // group-uniform
    if (__any_sync(full, need)) {
      if (need && g >= 0) {  // write the finished group's results
#pragma unroll
        for (int k = 0; k < TPL; k++) {
          const int64_t t = g * GT + gl * TPL + k;
          if (t >= P.n_targets) continue;
          if (res[k] >= BH_DROP) {
            push_resume(P, t, res[k], ax[k], ay[k], az[k], cnt[k], (!CONT && Li[k] < (res[k] & ~BH_DROP)) ? 1u : 0u);
          } else {
            if (!CONT) cnt[k] -= 1u;  // own record: "accepted", zero contribution
            wc += cnt[k];
            finish(P, load_target(P, t), (double)ax[k], (double)ay[k], (double)az[k], cnt[k]);
          }
        }
      }
      // one ticket per group that needs work.  The groups are split into one
      // contiguous Morton segment per SM; a warp takes tickets from its SM's
      // segment first (the warps resident on an SM then walk neighbouring
      // regions and share L1) and steals from the following segments after.
      int64_t mine = INT64_MAX;
      if (!PERSIST) {  // one group per group slot of the grid, no refill
        if (g < 0 && !first_done) mine = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GL;
        first_done = true;
      } else {
        const uint32_t m = __ballot_sync(full, need & (gl == 0));
        const int rank = __popc(m & lt);
        int left = __popc(m);
        int assigned = 0;
        while (left > 0 && hops < nseg) {
          const int64_t lo = ngroups * seg / nseg, hi = ngroups * (seg + 1) / nseg;
          uint32_t b = 0;
          if (lane == 0) b = atomicAdd(&P.st->sm_next[seg], (uint32_t)left);
          b = __shfl_sync(full, b, 0);
          const int64_t avail = hi - lo - (int64_t)b;
          const int take = avail <= 0 ? 0 : (avail < left ? (int)avail : left);
          if (rank >= assigned && rank < assigned + take) mine = lo + b + (rank - assigned);
          assigned += take;
          left -= take;
          if (left > 0) {
            seg = seg + 1 == nseg ? 0 : seg + 1;
            hops++;
          }
        }
      }
      const int64_t gnew = GL == 1 ? mine : __shfl_sync(full, mine, glead);
      if (need) {
        g = gnew;
        if (g >= ngroups) {
          parked = true;
          g = -1;
        } else {
#pragma unroll
          for (int k = 0; k < TPL; k++) {
            const int64_t t = g * GT + gl * TPL + k;
            float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t < P.n_targets) {
              const Target T = load_target(P, t);
              me = T.me;
              Li[k] = T.Li;
              res[k] = 0u;
            } else {
              res[k] = 0xffffffffu;
            }
            cnt[k] = 0;
            ax[k] = ay[k] = az[k] = 0.f;
            if (k & 1) {
              float lo, hi;
              up2(X[k >> 1], lo, hi);
              X[k >> 1] = pk2(lo, me.x);
              up2(Y[k >> 1], lo, hi);
              Y[k >> 1] = pk2(lo, me.y);
              up2(Z[k >> 1], lo, hi);
              Z[k >> 1] = pk2(lo, me.z);
            } else {
              X[k >> 1] = pk2(me.x, 0.f);
              Y[k >> 1] = pk2(me.y, 0.f);
              Z[k >> 1] = pk2(me.z, 0.f);
            }
          }
          c = 0;
        }
      }
      if (__all_sync(full, parked)) break;
    }
#pragma unroll 2
    for (int u = 0; u < BH_WALK2_UNROLL; u++) {
      const uint32_t cc = c;
      float4 cm;
      uint4 au;
      ld_rec(rec + cc, cm, au);
      const uint32_t skip = au.z;
      const float tacc = __uint_as_float(au.x), trej = __uint_as_float(au.y);
      uint32_t opn = 0u;
#pragma unroll
      for (int j = 0; j < NP; j++) {
        const int a = 2 * j, b = 2 * j + 1;
        const F2 DX = sub2(pk2(cm.x, cm.x), X[j]), DY = sub2(pk2(cm.y, cm.y), Y[j]),
                 DZ = sub2(pk2(cm.z, cm.z), Z[j]);
        const F2 D2 = fma2(DZ, DZ, fma2(DY, DY, mul2(DX, DX)));
        float d2A, d2B;
        up2(D2, d2A, d2B);
        float r2A, r2B;
        up2(add2(D2, E2), r2A, r2B);
        const F2 INV = pk2(rsqrt_fast(r2A), rsqrt_fast(r2B));
        float fA, fB;
        up2(mul2(mul2(pk2(cm.w, cm.w), mul2(INV, INV)), INV), fA, fB);
        if (CONT) {
          // a record containing the target is opened, never accepted (NaN
          // distance: every comparison is false)
          const bool cA = (cc <= Li[a]) & (skip > Li[a]), cB = (cc <= Li[b]) & (skip > Li[b]);
          const float qnan = __int_as_float(0x7fffffff);
          mac_pair(cc, cA ? qnan : d2A, cB ? qnan : d2B, tacc, trej, skip, res[a], res[b], cnt[a], cnt[b], opn, fA,
                   fB);
        } else {
          mac_pair(cc, d2A, d2B, tacc, trej, skip, res[a], res[b], cnt[a], cnt[b], opn, fA, fB);
        }
        const F2 FF = pk2(fA, fB);
        asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
            : "+f"(ax[a]), "+f"(ax[b]) : "l"(FF.v), "l"(DX.v));
        asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
            : "+f"(ay[a]), "+f"(ay[b]) : "l"(FF.v), "l"(DY.v));
        asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
            : "+f"(az[a]), "+f"(az[b]) : "l"(FF.v), "l"(DZ.v));
      }
      // the group descends if any of its targets opens; a group at the sentinel
      // (walk over, or parked: every res = ~0) stays there
      const bool go = GL == 1 ? opn != 0u : (__ballot_sync(full, opn != 0u) & gm) != 0u;
      c = min(go ? cc + 1u : skip, Wn);
    }
  }
  for (int o = 16; o; o >>= 1) wc += __shfl_xor_sync(full, wc, o);
  if (lane == 0 && wc) {
    atomicAdd(&P.st->interactions, wc);
    atomicAdd(&P.st->interactions_cum, wc);
  }
}

// Continuation of the targets that dropped out of the fast walk (k_walk_resume).
// One WARP per queued target.  A DFS segment (x, b) -- "visit x, then go on at
// skip(x) while below b" -- splits into x itself, the segment (x+1, skip(x)) of
// its subtree if x is opened, and the segment (skip(x), b) of what follows; the
// target's remaining walk is the segment (cdrop, Wn).  The warp pops up to 32
// segments from a LIFO in shared memory, each lane tests its node with the fp32
// filter (the oracle's fp64 formula, exact_accept, on inconclusive tests;
// records containing the target are opened, reading L5), interacts or pushes
// the subtree segment, and pushes the follow-on segment (ballot-ranked, so the
// order is deterministic).  Lane partials are fp64, reduced in lane order and
// added to the fast walk's fp32 prefix.  Queue slots beyond the resume-state
// capacity restart at (0, Wn) with zero partials.  A full stack (never seen;
// bounded by ~2 x 32 x depth) hands the remaining segments to lane 0, which
// walks each one stacklessly.
constexpr int RESUME_WARPS = 4;
#ifndef BH_RESUME_STACK_N
#define BH_RESUME_STACK_N 512
#endif
#ifndef BH_RESUME_MINB
#define BH_RESUME_MINB 8
#endif
constexpr int RESUME_STACK = BH_RESUME_STACK_N;

struct ResumeAcc {
  double ax, ay, az;
  uint32_t cnt, fb, nop;
};

// test node c for target T; returns true if accepted (and accumulates)
__device__ __forceinline__ bool resume_visit(const WalkParams &P, const Target &T, double Ld, uint32_t c,
                                             uint32_t &skip, ResumeAcc &A) {
  const float4 cm = P.rec[c].cm;
  const uint4 au = P.rec[c].aux;
  skip = au.z;
  const float dx = __fsub_rn(cm.x, T.me.x), dy = __fsub_rn(cm.y, T.me.y), dz = __fsub_rn(cm.z, T.me.z);
  const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
  const bool cont = (c <= T.Li) & (au.z > T.Li);
  bool acc = !cont & (d2 > __uint_as_float(au.x));
  if (!cont && !acc && d2 >= __uint_as_float(au.y)) {
    acc = exact_accept(P.rec_mom, c, au.w & META_LEVEL_MASK, T.me.x, T.me.y, T.me.z, Ld, P.theta2);
    A.fb++;
  }
  if (acc) {
    const float inv = rsqrt_fast(__fadd_rn(d2, P.eps2));
    const float f = __fmul_rn(__fmul_rn(cm.w, __fmul_rn(inv, inv)), inv);
    A.ax += (double)__fmul_rn(f, dx);
    A.ay += (double)__fmul_rn(f, dy);
    A.az += (double)__fmul_rn(f, dz);
    if (P.quad) {
      float qx = 0.f, qy = 0.f, qz = 0.f;
      quad_term(load_quad(P.qrec, c), dx, dy, dz, inv, true, qx, qy, qz);
      A.ax += (double)qx;
      A.ay += (double)qy;
      A.az += (double)qz;
    }
    A.cnt++;
  } else {
    A.nop++;
  }
  return acc;
}

__global__ void __launch_bounds__(32 * RESUME_WARPS, BH_RESUME_MINB) k_walk_resume(const WalkParams P) {
  __shared__ uint2 stack[RESUME_WARPS][RESUME_STACK];
  if (P.st->err & ERR_NODE_OVERFLOW) return;
  const uint32_t full = 0xffffffffu;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint2 *stk = stack[w];
  const uint32_t Wn = P.st->n_records;
  const unsigned long long nredo = P.st->n_redo;
  const double Ld = (double)P.st->L;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  for (unsigned long long k = blockIdx.x * (unsigned long long)RESUME_WARPS + w; k < nredo;
       k += (unsigned long long)gridDim.x * RESUME_WARPS) {
    const Target T = load_target(P, P.redo[k]);
    float pax = 0.f, pay = 0.f, paz = 0.f;
    uint32_t pcnt = 0, c0 = 0;
    if ((int64_t)k < P.cap_resume) {
      const ResumeState r = P.resume[k];
      pax = r.ax;
      pay = r.ay;
      paz = r.az;
      pcnt = r.cnt;
      c0 = r.cdrop;
    }
    ResumeAcc A = {0.0, 0.0, 0.0, 0u, 0u, 0u};
    uint32_t sp = 0;
    if (c0 < Wn) {
      if (lane == 0) stk[0] = make_uint2(c0, Wn);
      sp = 1;
    }
    bool overflow = false;
    __syncwarp();
    while (sp > 0 && !overflow) {
      const uint32_t nt = sp < 32u ? sp : 32u;
      const uint32_t base = sp - nt;
      const bool have = (uint32_t)lane < nt;
      const uint2 seg = have ? stk[base + lane] : make_uint2(0u, 0u);
      __syncwarp();
      sp = base;
      uint2 p1 = make_uint2(0u, 0u), p2 = make_uint2(0u, 0u);
      bool push1 = false, push2 = false;
      if (have) {
        uint32_t skip;
        const bool acc = resume_visit(P, T, Ld, seg.x, skip, A);
        push1 = skip < seg.y;                          // the follow-on segment
        p1 = make_uint2(skip, seg.y);
        push2 = !acc && seg.x + 1u < skip;             // the opened node's subtree
        p2 = make_uint2(seg.x + 1u, skip);
      }
      const uint32_t b1 = __ballot_sync(full, push1), b2 = __ballot_sync(full, push2);
      const uint32_t tot = __popc(b1) + __popc(b2);
      if (sp + tot > (uint32_t)P.resume_stack) {  // warp-uniform; lane 0 redoes the target below
        overflow = true;
        break;
      }
      // follow-on segments first (popped last), subtree segments on top: the
      // LIFO then goes depth-first
      if (push1) stk[sp + __popc(b1 & lt)] = p1;
      if (push2) stk[sp + __popc(b1) + __popc(b2 & lt)] = p2;
      sp += tot;
      __syncwarp();
    }
    // reduce the lane partials in lane order
    for (int o = 16; o; o >>= 1) {
      A.ax += __shfl_xor_sync(full, A.ax, o);
      A.ay += __shfl_xor_sync(full, A.ay, o);
      A.az += __shfl_xor_sync(full, A.az, o);
      A.cnt += __shfl_xor_sync(full, A.cnt, o);
      A.fb += __shfl_xor_sync(full, A.fb, o);
      A.nop += __shfl_xor_sync(full, A.nop, o);
    }
    if (overflow) {  // lane 0 walks the whole remaining segment stacklessly
      A = ResumeAcc{0.0, 0.0, 0.0, 0u, 0u, 0u};
      if (lane == 0) {
        uint32_t c = c0;
        while (c < Wn) {
          uint32_t skip;
          c = resume_visit(P, T, Ld, c, skip, A) ? skip : c + 1u;
        }
      }
    }
    if (lane == 0) {
      const uint32_t cnt = pcnt + A.cnt;
      atomicAdd(&P.st->interactions, (unsigned long long)cnt);
      atomicAdd(&P.st->interactions_cum, (unsigned long long)cnt);
      atomicAdd(&P.st->fallbacks, (unsigned long long)A.fb);
      atomicAdd(&P.st->opens, (unsigned long long)A.nop);
      atomicAdd(&P.st->opens_cum, (unsigned long long)A.nop);
      finish(P, T, (double)pax + A.ax, (double)pay + A.ay, (double)paz + A.az, cnt);
    }
    __syncwarp();
  }
}

cudaError_t launch_walk(const Workspace &W, const WalkArgs &a, cudaStream_t s) {
  if (a.n_targets <= 0) return cudaSuccess;
  WalkParams P;
  P.rec = W.rec;
  P.quad = a.quad && W.qrec;
  P.qrec = P.quad ? W.qrec : nullptr;
  P.rec_mom = W.rec_mom;
  P.nstart = W.nstart;
  P.vals = W.vals[a.buf];
  P.targets = W.targets;
  P.uid = W.uid;
  P.st = W.status;
  P.icount = W.icount;
  P.redo = W.redo;
  P.gcost = (!a.stats && !getenv("BH_NO_GROUP_ORDER")) ? W.gcost : nullptr;
  P.resume = W.resume;
  P.cap_resume = W.cap_resume;
  P.resume_stack = W.resume_stack > 0 && W.resume_stack < RESUME_STACK ? W.resume_stack : RESUME_STACK;
  P.need_cont = a.need_cont;
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
  P.num_sms = a.num_sms > 0 ? a.num_sms : 148;
  if (!a.stats && a.group >= 80 && a.group <= 95) {
    cudaError_t e = cudaMemsetAsync(W.status->sm_next, 0, sizeof(W.status->sm_next), s);
    if (e != cudaSuccess) return e;
  }
  unsigned grid = (unsigned)((a.n_targets + 255) / 256);
  if (!a.stats && a.group >= 80 && a.group <= 95) {
    // group walk (k_walk_lane): lanes per group x targets per lane
    //   80: 1 x 4   81: 1 x 2   82: 2 x 4   83: 2 x 2   84: 4 x 2   85: 4 x 4
    //   (persistent, SM-local tickets); +10: the same, one group per slot
    const bool cont = a.need_cont;
    const bool persist = a.group < 90;
    const int code = persist ? a.group : a.group - 10;
    cudaError_t e = cudaSuccess;
    int nb = 0, tpg = 4;
#define BH_LANE_CASE(code, GLv, NPv)                                                                 \
  case code:                                                                                          \
    tpg = GLv * 2 * NPv;                                                                              \
    e = cont ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_walk_lane<GLv, NPv, true, true>, 256, 0) \
             : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_walk_lane<GLv, NPv, false, true>, 256, 0); \
    break;
    switch (code) {
      BH_LANE_CASE(80, 1, 2)
      BH_LANE_CASE(81, 1, 1)
      BH_LANE_CASE(82, 2, 2)
      BH_LANE_CASE(83, 2, 1)
      BH_LANE_CASE(84, 4, 1)
      BH_LANE_CASE(85, 4, 2)
    }
#undef BH_LANE_CASE
    if (e != cudaSuccess) return e;
    if (nb < 1) nb = 1;
    const int64_t ngroups = (a.n_targets + tpg - 1) / tpg;
    const int lanes_per_group = code == 80 || code == 81 ? 1 : (code <= 83 ? 2 : 4);
    int64_t want = (ngroups * lanes_per_group + 255) / 256;  // no more threads than groups need
    int64_t gl = (int64_t)P.num_sms * nb;
    if (want < gl || !persist) gl = want;
    const unsigned gridl = (unsigned)(gl < 1 ? 1 : gl);
#define BH_LANE_LAUNCH(code, GLv, NPv)                                   \
  case code:                                                             \
    if (persist) {                                                       \
      if (cont) k_walk_lane<GLv, NPv, true, true><<<gridl, 256, 0, s>>>(P);  \
      else k_walk_lane<GLv, NPv, false, true><<<gridl, 256, 0, s>>>(P);      \
    } else {                                                             \
      if (cont) k_walk_lane<GLv, NPv, true, false><<<gridl, 256, 0, s>>>(P); \
      else k_walk_lane<GLv, NPv, false, false><<<gridl, 256, 0, s>>>(P);     \
    }                                                                    \
    break;
    switch (code) {
      BH_LANE_LAUNCH(80, 1, 2)
      BH_LANE_LAUNCH(81, 1, 1)
      BH_LANE_LAUNCH(82, 2, 2)
      BH_LANE_LAUNCH(83, 2, 1)
      BH_LANE_LAUNCH(84, 4, 1)
      BH_LANE_LAUNCH(85, 4, 2)
    }
#undef BH_LANE_LAUNCH
  } else if (!a.stats && (a.group == 0 || a.group >= 64)) {
    // production path (k_walk2): packed fp32, lanes per group x targets per lane
    //   66 / 67 / 68: 8 / 4 / 2 lanes x 2 targets   (api.cu picks 67 or 68 for 0)
    //   64: 32 lanes x 2 targets;  65 / 69 / 70: 8 / 4 / 2 lanes x 4 targets
    const bool cont = a.need_cont;
    constexpr int WB = BH_WALK2_BLOCK;
    const unsigned grid2 = (unsigned)((a.n_targets + 2 * WB - 1) / (2 * WB));
    const unsigned g4 = (unsigned)((a.n_targets + 4 * WB - 1) / (4 * WB));
#define BH_WALK2_LAUNCH(GLv, NPv, gr)                                              \
  if (P.quad) {                                                                   \
    if (cont) k_walk2<GLv, NPv, true, true><<<gr, WB, 0, s>>>(P);                \
    else k_walk2<GLv, NPv, false, true><<<gr, WB, 0, s>>>(P);                    \
  } else {                                                                        \
    if (cont) k_walk2<GLv, NPv, true, false><<<gr, WB, 0, s>>>(P);               \
    else k_walk2<GLv, NPv, false, false><<<gr, WB, 0, s>>>(P);                   \
  }
    switch (a.group) {
      case 64: BH_WALK2_LAUNCH(32, 1, grid2) break;
      case 65: BH_WALK2_LAUNCH(8, 2, g4) break;
      case 66: BH_WALK2_LAUNCH(8, 1, grid2) break;
      case 68: BH_WALK2_LAUNCH(2, 1, grid2) break;
      case 69: BH_WALK2_LAUNCH(4, 2, g4) break;
      case 70: BH_WALK2_LAUNCH(2, 2, g4) break;
      default: BH_WALK2_LAUNCH(4, 1, grid2) break;  // 67
    }
#undef BH_WALK2_LAUNCH
  } else {
#define BH_WALK_CASE(g)                                                     \
  case g:                                                                   \
    if (a.stats) k_walk<g, true><<<grid, 256, 0, s>>>(P);                   \
    else k_walk<g, false><<<grid, 256, 0, s>>>(P);                          \
    break;
  switch (a.group) {
    BH_WALK_CASE(1)
    BH_WALK_CASE(2)
    BH_WALK_CASE(4)
    BH_WALK_CASE(8)
    BH_WALK_CASE(16)
    default:
    BH_WALK_CASE(32)
  }
#undef BH_WALK_CASE
  }
  // the continuation of dropped-out targets: a fixed grid, grid-stride over the
  // device-side queue (lanes dense in queue order)
  int64_t eg = (a.n_targets + RESUME_WARPS - 1) / RESUME_WARPS;
  if (eg > 148 * 16) eg = 148 * 16;
  k_walk_resume<<<(unsigned)eg, 32 * RESUME_WARPS, 0, s>>>(P);
  return cudaGetLastError();
}

}  // namespace bh
