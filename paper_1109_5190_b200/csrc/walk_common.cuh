// walk_common.cuh -- what the K6 walk kernels share: the launch parameters,
// target load / epilogue (K7 fused leapfrog) / drop-out queue, the quadrupole
// term and the packed-fp32 (f32x2) helpers.
//   walk.cu          k_walk (production, every group size) and launch_walk
//   walk_resume.cu   k_walk_resume (continuation of inconclusive MAC tests, fp64)
//
// PAPER.md:500-504 (§3): "The most computationally intensive part of the
// Barnes-Hut algorithm is the force computation stage."  PAPER.md:408-415:
// a remote cluster is treated as a single body only if D > r/theta.  Readings
// (DESIGN.md §3): r = cell side s_l = L 2^-l (L1), D = distance to the centre
// of mass (L2), strict s^2 < theta^2 D^2 (L3, L4), cells containing the target
// are always opened (L5), Plummer softening on every source (L6), G applied
// last (L7); "interactions" = accepted cells + particles j != i (L21).
//
// Per-particle semantics with shared traversal.  Targets are
// taken in Morton order; a group of GL lanes (2 GL targets) walks ONE
// stackless DFS over the record array: at record c every active target
// evaluates its own MAC; targets that accept c interact with it and become
// inactive until skip(c) (their subtree is done); the group descends (c + 1) if
// any active target opens c, else jumps to skip(c).  Each target therefore
// sees exactly its own Barnes-Hut frontier, in DFS order -- identical
// decisions to the oracle's recursive walk -- while the group's record loads
// are one broadcast address.
//
// MAC decisions are exact.  The fast kernel decides with the fp32 thresholds
// T_acc / T_rej of com.cu (d2_32 > T_acc: accept for sure; d2_32 < T_rej: open
// for sure).  A target whose d2_32 falls between them (~1e-6 of the tests)
// drops out of the fast walk at that record and is queued with its partial
// sums; k_walk_resume then continues each such target's DFS from that record
// alone, with the oracle's fp64 test on the ambiguous nodes.
//
// Interaction (fp32): r2 = d2 + eps^2, f = M rsqrt(r2)^3, a += f (dx, dy, dz):
// 18 flops + 1 MUFU.RSQ, in the target's own DFS order; the fp32 sums run over
// blocks of BH_FOLD_TRIPS loop trips of the group's walk and are folded into
// an outer sum (walk.cu; measured max error over all 2^24 cfg4 targets 1.3e-4
// with one fp32 sum, 1.5e-5 with the fold).
//
// K7 (mode 1): v += a * kick (kick = dt/2 on the first step, dt after; reading
// L8), x += v dt, written in place to pos4 / vel4 of the particle's storage slot
// (the walk reads positions from the records, never from pos4).
#pragma once

#include <math.h>
#include <stdlib.h>

#include "bh_internal.cuh"

namespace bh {

struct WalkParams {
  const Rec *__restrict__ rec;
  const float4 *__restrict__ qrec;  // multipole = 2: -Q (fp32) per record, 2 float4 (else null)
  int quad;
  const double4 *__restrict__ lvl_mom;   // fp64 moments of the level items (exact MAC)
  const uint32_t *__restrict__ rec_item;  // record -> level item
  const uint32_t *__restrict__ nstart;
  const uint32_t *__restrict__ vals;
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
  uint32_t *gcost;  // group-order cost per storage id: the loop trips of its group's last walk (or null)
  int user_order;
  int64_t n_targets;   // all particles (targets are sorted positions 0 .. n-1)
  // world > 1: the walk runs the P = 1 groups (GT consecutive sorted
  // positions) that hold at least one own particle -- group_list[0 ..
  // *n_groups_dev) -- and writes only the own targets' results, so every
  // target is summed in the same group, hence the same blocks, as at P = 1
  const uint32_t *group_list;
  const uint32_t *n_groups_dev;
  int own_check;
  int mode;
  float eps2, G, kick, dt;
  double theta2;
  uint32_t own_lo, own_hi;
  int num_sms;
  // fused exchange (bh_set_peers): every other rank's pos4 replica, written
  // by K7 beside the own copy (peer memory over NVLink)
  int n_peers;
  float4 *peer_pos4[BH_MAX_PEERS];
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

struct Target {
  uint32_t p, Li, s;
  float4 me;
};

__device__ __forceinline__ Target load_target(const WalkParams &P, int64_t t) {
  Target T;
  T.p = (uint32_t)t;  // a sorted position
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
    const float4 x = make_float4(fmaf(v.x, P.dt, T.me.x), fmaf(v.y, P.dt, T.me.y), fmaf(v.z, P.dt, T.me.z), T.me.w);
    P.pos4[T.s] = x;
    // K8 fused into K7 (bh_set_peers): the new position goes straight into
    // every other rank's replica, so the exchange rides on the walk
    for (int k = 0; k < P.n_peers; k++) P.peer_pos4[k][T.s] = x;
  }
}

// A target whose fp32 MAC test was inconclusive at record cdrop (its resume
// word is BH_DROP | cdrop) is queued with its fp32 partial sums and count over
// the DFS prefix before cdrop; k_walk_resume continues the same DFS from
// cdrop with the oracle's exact test.  `own` = 1 if the count includes the
// target's own record (the CONT = false kernels accept it with a zero
// contribution; the resume kernel opens it, as the oracle does).
__device__ __forceinline__ void push_resume(const WalkParams &P, int64_t t, uint32_t res, double ax, double ay,
                                            double az, uint32_t cnt, uint32_t own) {
  const unsigned long long k = atomicAdd(&P.st->n_redo, 1ull);
  P.redo[k] = (uint32_t)t;
  if ((int64_t)k < P.cap_resume) {
    ResumeState r;
    r.ax = ax;
    r.ay = ay;
    r.az = az;
    r.cnt = cnt - own;
    r.cdrop = res & ~BH_DROP;
    P.resume[k] = r;
  }
}

// ---------------------------------------------------------------- packed fp32
// Blackwell's packed fp32 instructions (FADD2 / FMUL2 / FFMA2: one issue slot,
// two fp32 results), used by k_walk to carry two targets per lane.
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

// one record, one 32-byte load (measured r2: the record split into two 16-B
// arrays -- two loads per visit -- cost cfg4 +37 %, cfg5 +43 % walk time)
__device__ __forceinline__ void ld_rec(const Rec *p, float4 &cm, uint4 &au) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(cm.x), "=f"(cm.y), "=f"(cm.z), "=f"(cm.w), "=r"(au.x), "=r"(au.y), "=r"(au.z), "=r"(au.w)
               : "l"(p));
}

// k_walk_resume geometry (walk_resume.cu; launch_walk clamps the stack-depth
// test hook to RESUME_STACK)
constexpr int RESUME_WARPS = 4;
#ifndef BH_RESUME_STACK_N
#define BH_RESUME_STACK_N 512
#endif
#ifndef BH_RESUME_MINB
#define BH_RESUME_MINB 8
#endif
constexpr int RESUME_STACK = BH_RESUME_STACK_N;

void launch_walk_resume(const WalkParams &P, int64_t n_targets, cudaStream_t s);

// level of record c: its level-ordered item's level (levels 0 .. 22, 22 =
// bucket member), from the level offsets of K4
__device__ __forceinline__ uint32_t record_level(const WalkParams &P, uint32_t c) {
  const uint32_t it = P.rec_item[c];
  uint32_t l = 0;
#pragma unroll 1
  while (l + 1 < BH_NLEVELS && P.st->lvl_offset[l + 1] <= it) l++;
  return l;
}

}  // namespace bh
