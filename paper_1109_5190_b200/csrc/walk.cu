// walk.cu -- K6 force walk (+ K7 fused leapfrog): the production kernel
// k_walk2 and launch_walk.  Semantics, readings and the shared pieces:
// walk_common.cuh.
#include "walk_common.cuh"

namespace bh {

// ---------------------------------------------------------------- k_walk2
// The production walk: the same per-lane semantics and the same fp32 operation
// sequence per target as k_walk (bitwise-identical results), but every lane
// carries TWO targets and does their arithmetic with Blackwell's packed fp32
// instructions (FADD2 / FMUL2 / FFMA2: one issue slot, two fp32 results; the
// node's fields enter as broadcast scalar operands).  The record loads, the
// traversal control and the vote are shared by the pair, so the issue slots per
// target-visit drop by ~1/3.  A group of GL lanes (2 GL targets, Morton-
// consecutive) shares one traversal.
#ifndef BH_WALK2_BLOCK
#define BH_WALK2_BLOCK 128
#endif
#ifndef BH_WALK2_UNROLL_SMALL
#define BH_WALK2_UNROLL_SMALL 3  // visits per loop trip for groups of <= 2 lanes (3 vs 2: cfg5 -2.2%, cfg3 -1.2%, cfg2 -1.4%)
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
   for (int u = 0; u < (GL <= 2 ? BH_WALK2_UNROLL_SMALL : BH_WALK2_UNROLL); u++) {
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

cudaError_t launch_walk(const Workspace &W, const WalkArgs &a, cudaStream_t s) {
  if (a.n_targets <= 0) return cudaSuccess;
  WalkParams P;
  P.rec = W.rec;
  P.quad = a.quad && W.qrec;
  P.qrec = P.quad ? W.qrec : nullptr;
  P.lvl_mom = W.lvl_mom;
  P.rec_item = W.rec_item;
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
    const cudaError_t e = launch_walk_lane(P, a.group, a.need_cont, a.n_targets, s);
    if (e != cudaSuccess) return e;
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
    launch_walk_simple(P, a.group, a.stats, a.n_targets, s);
  }
  launch_walk_resume(P, a.n_targets, s);
  return cudaGetLastError();
}

}  // namespace bh
