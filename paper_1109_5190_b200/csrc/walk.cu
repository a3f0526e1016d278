// walk.cu -- K6 force walk (+ K7 fused leapfrog): k_walk and launch_walk.
// Semantics, readings and the shared pieces: walk_common.cuh.
//
// Every lane carries TWO targets and evaluates them with Blackwell's packed
// fp32 instructions (FADD2 / FMUL2 / FFMA2: one issue slot, two fp32 results;
// the record's fields enter as broadcast scalar operands).  A group of GL
// lanes (2 GL Morton-consecutive targets) shares one stackless traversal; the
// record load, the traversal control and the vote are shared by the group.
//
// Per target and record visit the MAC costs 7 ALU-pipe instructions (the loop
// is ALU-pipe bound): act = c >= res (ISETP), acc = act & d2 >
// T_acc, ge = act & d2 >= T_rej (2 FSETP), cnt += acc, f = acc ? f : 0,
// res = ge ? (acc ? skip : dropw) : res (2 SEL).  The record's fourth word is
// its drop word (BH_DROP | c, so the inconclusive case needs no per-visit OR);
// a target opens c iff its updated res <= c (accept and drop move res past c,
// inactive targets are past it already), so the group vote is one min per
// lane.  The sentinel record Wn (T_acc = +inf, T_rej = -inf, skip = Wn, drop
// word Wn + 1) parks finished groups: its targets go inactive without a drop
// and nobody opens it, so the cursor never passes Wn and needs no clamp.
//
// 4 targets per lane (NP = 2, the large configurations) use the leanest form
// (MR2): the MAC filter compares the softened r2 (BH_EPS_FOLD, com.cu), runs
// before the rsqrt and replaces r2 by +inf for a target that does not accept
// (rsqrt(+inf) = 0: no force, no mask multiply); the accept count stays a
// float flag summed per pair, except for a lane's own group (GL = 1), which
// sums rsqrt(r2m)^2 x r2 on the FMA pipe (1 +- 2^-20 or exactly 0, rounded to
// the integer at every flush) and so spends 5 ALU-pipe instructions per
// target and visit: ISETP, 2 FSETP, SEL (res), FSEL (r2m).
#include "walk_common.cuh"

namespace bh {

#ifndef BH_WALK_BLOCK
#define BH_WALK_BLOCK 128
#endif
#ifndef BH_WALK_MINB
#define BH_WALK_MINB 9  // blocks of 128 threads per SM: 56 registers (36 warps; 10 spills in the loop)
#endif
#ifndef BH_WALK_UNROLL
#define BH_WALK_UNROLL 2  // record visits per loop trip, groups of >= 4 lanes
#endif
#ifndef BH_WALK_UNROLL_NP2
#define BH_WALK_UNROLL_NP2 4  // 4 targets per lane (4 vs 3, with 32-trip blocks: cfg4 walk 38.05 -> 37.75 ms, cfg5 63.99 -> 63.13)
#endif
#ifndef BH_WALK_UNROLL_SMALL
#define BH_WALK_UNROLL_SMALL 4  // groups of <= 2 lanes, 2 targets per lane (3 vs 2: cfg5 -2.2%, cfg3 -1.2%, cfg2 -1.4%, r1; 4 vs 3: cfg2 -1.3%, r2zf)
#endif
#ifndef BH_WALK_UNROLL_NP2_L1
#define BH_WALK_UNROLL_NP2_L1 5  // a lane's own 4 targets (code 70; 5 vs 4: cfg5 walk 63.15 -> 62.85 ms; code 69 lost 9% at 5)
#endif
// Accumulation: every target's contributions are summed in fp32 over blocks
// of BH_FOLD_TRIPS loop trips of its group's walk, and each block is folded
// into an outer sum: fold mode 1 = fp32 outer sums in registers (NP = 1),
// 3 = fp32 outer sums in shared memory (NP = 2, whose registers are full),
// 2 = fp64 in registers, 0 = one fp32 sum.  The trip counter is uniform over
// the warp (a non-divergent branch), and the blocks -- hence the rounding --
// depend only on the group's own walk (the same at any rank count: world > 1
// walks the P = 1 groups).  Measured on all 2^24 cfg4 targets
// (profiles/r2_summary.md): max relative error 1.26e-4 with one fp32 sum,
// 1.45e-5 with fp32 block sums (8-target groups of 4 lanes x 2), 2.2e-5
// (2 lanes x 4), 6.5e-6 with fp64 outer sums.
#ifndef BH_FOLD
#define BH_FOLD 1      // NP = 1 (0 / 1 / 2)
#endif
#ifndef BH_FOLD_NP2
#define BH_FOLD_NP2 3  // NP = 2 (0 / 1 / 3)
#endif
#ifndef BH_RSQRT_NEWTON
#define BH_RSQRT_NEWTON 0
#endif
#ifndef BH_FOLD_TRIPS
#define BH_FOLD_TRIPS 32  // (16 before r2z; 32 measured: cfg4 max error 1.6e-5, cfg5 6.7e-5 -- its per-term floor)
#endif
#ifndef BH_WALK_MINB2
#define BH_WALK_MINB2 7  // NP = 2 (4 targets per lane): 72 registers, no spill in the loop (8 blocks: 64, cfg4 +4.5%)
#endif
template <int FM> struct FoldType { typedef float T; };
template <> struct FoldType<2> { typedef double T; };

// One target's MAC at record cc (see the header comment); with QUAD the
// quadrupole factors of a target that does not accept are zeroed too.
template <bool QUAD>
__device__ __forceinline__ void mac_one(uint32_t cc, float d2, float tacc, float trej, uint32_t skip, uint32_t dropw,
                                        uint32_t &res, uint32_t &cnt, float &f, float &g1, float &g2) {
  if (QUAD) {
    asm("{\n\t.reg .pred pa, pc, pq;\n\t"
        "setp.ge.u32 pa, %5, %0;\n\t"
        "setp.gt.and.f32 pc, %6, %7, pa;\n\t"
        "setp.ge.and.f32 pq, %6, %8, pa;\n\t"
        "@pc add.u32 %1, %1, 1;\n\t"
        "@pq selp.b32 %0, %9, %10, pc;\n\t"
        "@!pc mov.b32 %2, 0f00000000;\n\t"
        "@!pc mov.b32 %3, 0f00000000;\n\t"
        "@!pc mov.b32 %4, 0f00000000;\n\t}"
        : "+r"(res), "+r"(cnt), "+f"(f), "+f"(g1), "+f"(g2)
        : "r"(cc), "f"(d2), "f"(tacc), "f"(trej), "r"(skip), "r"(dropw));
  } else {
    asm("{\n\t.reg .pred pa, pc, pq;\n\t"
        "setp.ge.u32 pa, %3, %0;\n\t"
        "setp.gt.and.f32 pc, %4, %5, pa;\n\t"
        "setp.ge.and.f32 pq, %4, %6, pa;\n\t"
        "@pc add.u32 %1, %1, 1;\n\t"
        "@pq selp.b32 %0, %7, %8, pc;\n\t"
        "@!pc mov.b32 %2, 0f00000000;\n\t}"
        : "+r"(res), "+r"(cnt), "+f"(f)
        : "r"(cc), "f"(d2), "f"(tacc), "f"(trej), "r"(skip), "r"(dropw));
  }
}

// The same decision without a predicate left alive: res is updated in place
// and the accept flag comes back as a float (1 or 0) that masks the force and
// is summed as the count on the FMA pipe (packed, per pair).  Used where the
// unmasked force is finite for every record (eps > 0 and no NaN distance:
// the kernels without the containment test), so 0 x f = 0.
__device__ __forceinline__ void mac_accf(uint32_t cc, float d2, float tacc, float trej, uint32_t skip, uint32_t dropw,
                                         uint32_t &res, float &accf) {
  asm("{\n\t.reg .pred pa, pc, pq;\n\t"
      "setp.ge.u32 pa, %2, %0;\n\t"
      "setp.gt.and.f32 pc, %3, %4, pa;\n\t"
      "setp.ge.and.f32 pq, %3, %5, pa;\n\t"
      "@pq selp.b32 %0, %6, %7, pc;\n\t"
      "selp.f32 %1, 0f3F800000, 0f00000000, pc;\n\t}"
      : "+r"(res), "=f"(accf)
      : "r"(cc), "f"(d2), "f"(tacc), "f"(trej), "r"(skip), "r"(dropw));
}

// BH_MASK_R2: the same, and r2 replaced by +inf for a target that does not
// accept (rsqrt(+inf) = 0: the force vanishes without the mask multiply)
__device__ __forceinline__ void mac_accf_r2(uint32_t cc, float d2, float tacc, float trej, uint32_t skip,
                                            uint32_t dropw, uint32_t &res, float &accf, float &r2m) {
  asm("{\n\t.reg .pred pa, pc, pq;\n\t"
      "setp.ge.u32 pa, %3, %0;\n\t"
      "setp.gt.and.f32 pc, %4, %5, pa;\n\t"
      "setp.ge.and.f32 pq, %4, %6, pa;\n\t"
      "@pq selp.b32 %0, %7, %8, pc;\n\t"
      "selp.f32 %1, 0f3F800000, 0f00000000, pc;\n\t"
      "selp.f32 %2, %4, 0f7F800000, pc;\n\t}"
      : "+r"(res), "=f"(accf), "=f"(r2m)
      : "r"(cc), "f"(d2), "f"(tacc), "f"(trej), "r"(skip), "r"(dropw));
}
// (2 = for 4 targets per lane only: cfg4 walk 39.5 -> 38.2 ms, cfg5 66.0 -> 65.3,
// cfg3 0.705 -> 0.690; 2 targets per lane lost, cfg2 0.605 -> 0.623)
// ... and no flag at all: the count is summed as rsqrt(r2m)^2 x r2 on the FMA
// pipe (BH_MR2_FCNT: 1 +- 2^-20 for an accept, exactly 0 otherwise; rounded
// to the integer at every flush, <= 160 terms per block: error < 2e-3)
__device__ __forceinline__ void mac_r2(uint32_t cc, float d2, float tacc, float trej, uint32_t skip,
                                       uint32_t dropw, uint32_t &res, float &r2m) {
  asm("{\n\t.reg .pred pa, pc, pq;\n\t"
      "setp.ge.u32 pa, %2, %0;\n\t"
      "setp.gt.and.f32 pc, %3, %4, pa;\n\t"
      "setp.ge.and.f32 pq, %3, %5, pa;\n\t"
      "@pq selp.b32 %0, %6, %7, pc;\n\t"
      "selp.f32 %1, %3, 0f7F800000, pc;\n\t}"
      : "+r"(res), "=f"(r2m)
      : "r"(cc), "f"(d2), "f"(tacc), "f"(trej), "r"(skip), "r"(dropw));
}
// (2 = a lane's own group only: cfg5 walk 65.31 -> 65.03 ms; with 2-lane
// groups it lost, cfg4 38.19 -> 38.64, though it issues 63 instead of 66
// instructions per visit: the FMA pipe, not issue, binds there)
#ifndef BH_MR2_FCNT
#define BH_MR2_FCNT 2
#endif
// (an integer count by a predicated add instead was measured: ptxas
// materialises the predicates, 74 vs 66 instructions per visit)
#ifndef BH_MASK_R2
#define BH_MASK_R2 2
#endif

// STATS: also count the opened MAC tests (the flop model of bench.py).
template <int GL, int NP, bool CONT, bool QUAD, bool STATS>
__global__ void __launch_bounds__(BH_WALK_BLOCK, QUAD ? 8 : (NP == 1 ? BH_WALK_MINB : BH_WALK_MINB2)) k_walk(const WalkParams P) {
  constexpr int TPL = 2 * NP;              // targets per lane (NP packed pairs)
  // the force mask on r2 (BH_MASK_R2, 4 targets per lane by default)
  constexpr bool MR2 = (BH_MASK_R2 == 1 || (BH_MASK_R2 == 2 && NP == 2)) && BH_EPS_FOLD && !CONT && !QUAD;
  constexpr bool MFC = MR2 && (BH_MR2_FCNT == 1 || (BH_MR2_FCNT == 2 && GL == 1));  // count = rsqrt^2 x r2
  constexpr bool FCNT = !CONT;  // float accept counts, flushed every BH_FOLD_TRIPS  // float accept counts (flushed every BH_FOLD_TRIPS)
  constexpr int GT = GL * TPL;             // targets per group
  constexpr int GPB = BH_WALK_BLOCK / GL;  // groups per block
  const uint32_t full = 0xffffffffu;
  if (P.st->err & ERR_NODE_OVERFLOW) return;
  const uint32_t Wn = P.st->n_records;
  const int lane = threadIdx.x & 31;
  const uint32_t gmask = GL == 32 ? full : (((1u << GL) - 1u) << (lane & ~(GL - 1)));
  const int64_t ngroups = P.group_list ? (int64_t)*P.n_groups_dev : (P.n_targets + GT - 1) / GT;
  const int64_t g0 = (int64_t)blockIdx.x * GPB;
  if (g0 >= ngroups) return;  // (world > 1: the grid is sized for the most groups a rank can hold)
  // Group order.  The block's groups are dealt to its warps in descending
  // order of their predicted cost (the loop trips of the group's last walk,
  // kept per particle in gcost so that it follows the particles as groups
  // re-form every step; a group's cost = the larger of its first and last
  // targets'): a warp runs until its slowest group is done, so warps of
  // similar groups idle less.  Which targets walk together does not change,
  // hence neither do the results.  Without costs: Morton order.
  const int gi = lane / GL, gl = lane % GL;
  int lg = (threadIdx.x >> 5) * (32 / GL) + gi;
  if (P.gcost) {
    __shared__ uint32_t s_cost[GPB], s_perm[GPB];
    if (threadIdx.x < GPB) {
      uint32_t cst = 0u;
      const int64_t g = g0 + threadIdx.x;
      if (g < ngroups) {
        const int64_t t0 = (P.group_list ? (int64_t)P.group_list[g] : g) * GT;
        const int64_t t1 = min(t0 + GT, P.n_targets) - 1;
        cst = max(P.gcost[P.vals[t0]], P.gcost[P.vals[t1]]);
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
  const int64_t gidx = g0 + lg;
  const bool gin = gidx < ngroups;
  const int64_t grp = gin ? (P.group_list ? (int64_t)P.group_list[gidx] : gidx) : 0;
  const int64_t tbase = grp * GT + gl;
  // the targets' positions (and, with CONT, own records) for the loop; the
  // rest of a target is re-read after the loop (not kept live across it)
  uint32_t res[TPL], cnt[TPL], nop[TPL];
  uint32_t sv_rec = 0, sv_leaf = 0;  // STATS: record loads, of particle records
  F2 CNT[NP];  // !CONT: per-pair fp32 accept counts, flushed into cnt every BH_FOLD_TRIPS trips
  float ax[TPL], ay[TPL], az[TPL];
  F2 X[NP], Y[NP], Z[NP];
  uint32_t Li[TPL];
  bool anyv = false;
  {
    Target T[TPL];
    bool v[TPL];
#pragma unroll
    for (int k = 0; k < TPL; k++) {
      const int64_t t = tbase + (int64_t)k * GL;
      v[k] = gin && t < P.n_targets;
      anyv |= v[k];
      if (v[k]) T[k] = load_target(P, t);
      else { T[k].p = 0; T[k].Li = 0; T[k].s = 0; T[k].me = make_float4(0.f, 0.f, 0.f, 0.f); }
      res[k] = v[k] ? 0u : 0xffffffffu;
      cnt[k] = 0;
      nop[k] = 0;
      ax[k] = ay[k] = az[k] = 0.f;
      Li[k] = T[k].Li;
    }
#pragma unroll
    for (int j = 0; j < NP; j++) {
      CNT[j] = pk2(0.f, 0.f);
      X[j] = pk2(T[2 * j].me.x, T[2 * j + 1].me.x);
      Y[j] = pk2(T[2 * j].me.y, T[2 * j + 1].me.y);
      Z[j] = pk2(T[2 * j].me.z, T[2 * j + 1].me.z);
    }
  }
  const F2 E2 = pk2(P.eps2, P.eps2);
  const bool gvalid = (__ballot_sync(full, anyv) & gmask) != 0u;
  const Rec *__restrict__ rec = P.rec;
  uint32_t gmask2 = gmask;
  asm volatile("" : "+r"(gmask2));  // a plain register: the group test is one LOP3
  uint32_t c = gvalid ? 0u : Wn;
  uint32_t git = 0;  // live loop trips of this lane's group (its cost; visits per trip = the unroll)
  constexpr int FM = NP == 1 ? BH_FOLD : BH_FOLD_NP2;  // fold mode
  typedef typename FoldType<FM>::T FoldT;
  // FM 1 / 2: the outer sums in registers; FM 3: in shared memory, [3 TPL][BLOCK]
  FoldT ox[FM == 1 || FM == 2 ? TPL : 1], oy[FM == 1 || FM == 2 ? TPL : 1], oz[FM == 1 || FM == 2 ? TPL : 1];
  __shared__ float s_out[FM == 3 ? 3 * TPL : 1][FM == 3 ? BH_WALK_BLOCK : 1];
  // FM 3 also keeps the flushed integer counts in shared memory (no registers)
  __shared__ uint32_t s_cnt[FM == 3 ? TPL : 1][FM == 3 ? BH_WALK_BLOCK : 1];
  if constexpr (FM == 1 || FM == 2) {
#pragma unroll
    for (int k = 0; k < TPL; k++) ox[k] = oy[k] = oz[k] = (FoldT)0;
  }
  if constexpr (FM == 3) {
#pragma unroll
    for (int k = 0; k < 3 * TPL; k++) s_out[k][threadIdx.x] = 0.f;
#pragma unroll
    for (int k = 0; k < TPL; k++) s_cnt[k][threadIdx.x] = 0u;
  }
  uint32_t trip = 0;
  if (__any_sync(full, c < Wn)) for (;;) {
#pragma unroll
    for (int u = 0; u < (NP == 2 ? (GL == 1 ? BH_WALK_UNROLL_NP2_L1 : BH_WALK_UNROLL_NP2)
                                 : GL <= 2 ? BH_WALK_UNROLL_SMALL : BH_WALK_UNROLL); u++) {
      const uint32_t cc = c;
      float4 cm;
      uint4 au;
      ld_rec(rec + cc, cm, au);
      const uint32_t skip = au.z, dropw = au.w;
      const float tacc = __uint_as_float(au.x), trej = __uint_as_float(au.y);
#pragma unroll
      for (int j = 0; j < NP; j++) {
        const int ka = 2 * j, kb = 2 * j + 1;
        const F2 DX = sub2(pk2(cm.x, cm.x), X[j]), DY = sub2(pk2(cm.y, cm.y), Y[j]), DZ = sub2(pk2(cm.z, cm.z), Z[j]);
#if BH_EPS_FOLD
        // the softened distance, which the MAC filter compares too (com.cu)
        const F2 R2 = fma2(DZ, DZ, fma2(DY, DY, fma2(DX, DX, E2)));
        float r2A, r2B;
        up2(R2, r2A, r2B);
        const float d2A = r2A, d2B = r2B;
#else
        const F2 D2 = fma2(DZ, DZ, fma2(DY, DY, mul2(DX, DX)));
        float d2A, d2B;
        up2(D2, d2A, d2B);
        float r2A, r2B;
        const F2 R2 = add2(D2, E2);
        up2(R2, r2A, r2B);
#endif
        if constexpr (MR2) {
          // the MAC first; a target that does not accept gets r2 = +inf, so
          // its rsqrt and force are 0 (no mask multiply)
          float rmA, rmB;
          if constexpr (MFC) {
            mac_r2(cc, r2A, tacc, trej, skip, dropw, res[ka], rmA);
            mac_r2(cc, r2B, tacc, trej, skip, dropw, res[kb], rmB);
          } else {
            float accA, accB;
            mac_accf_r2(cc, r2A, tacc, trej, skip, dropw, res[ka], accA, rmA);
            mac_accf_r2(cc, r2B, tacc, trej, skip, dropw, res[kb], accB, rmB);
            CNT[j] = add2(CNT[j], pk2(accA, accB));
          }
          const F2 INV = pk2(rsqrt_fast(rmA), rsqrt_fast(rmB));
          const F2 INV2 = mul2(INV, INV);
          if constexpr (MFC) CNT[j] = fma2(INV2, R2, CNT[j]);
          const F2 FF = mul2(mul2(pk2(cm.w, cm.w), INV2), INV);
          asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
              : "+f"(ax[ka]), "+f"(ax[kb]) : "l"(FF.v), "l"(DX.v));
          asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
              : "+f"(ay[ka]), "+f"(ay[kb]) : "l"(FF.v), "l"(DY.v));
          asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
              : "+f"(az[ka]), "+f"(az[kb]) : "l"(FF.v), "l"(DZ.v));
          continue;
        }
        // the interaction of both targets, branch-free (f zeroed for a target
        // that does not accept the record)
#if BH_RSQRT_NEWTON
        // (accuracy experiment: one Newton step on MUFU.RSQ, y (1.5 - 0.5 r2 y^2))
        F2 INV = pk2(rsqrt_fast(r2A), rsqrt_fast(r2B));
        {
          const F2 H = fma2(pk2(-0.5f, -0.5f), mul2(mul2(R2, INV), INV), pk2(1.5f, 1.5f));
          INV = mul2(INV, H);
        }
#else
        const F2 INV = pk2(rsqrt_fast(r2A), rsqrt_fast(r2B));
#endif
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
        // per-target MAC; a record containing the target is opened, never
        // accepted (CONT: NaN distance)
        float qA = d2A, qB = d2B;
        if (CONT) {
          const bool cA = (cc <= Li[ka]) & (skip > Li[ka]), cB = (cc <= Li[kb]) & (skip > Li[kb]);
          const float qnan = __int_as_float(0x7fffffff);
          qA = cA ? qnan : d2A;
          qB = cB ? qnan : d2B;
        }
        F2 FF;
        if (CONT) {
          mac_one<QUAD>(cc, qA, tacc, trej, skip, dropw, res[ka], cnt[ka], fA, g1A, g2A);
          mac_one<QUAD>(cc, qB, tacc, trej, skip, dropw, res[kb], cnt[kb], fB, g1B, g2B);
          FF = pk2(fA, fB);
        } else {
          float accA, accB;
          mac_accf(cc, qA, tacc, trej, skip, dropw, res[ka], accA);
          mac_accf(cc, qB, tacc, trej, skip, dropw, res[kb], accB);
          const F2 ACC = pk2(accA, accB);
          FF = mul2(pk2(fA, fB), ACC);
          CNT[j] = add2(CNT[j], ACC);
          if (QUAD) {
            float ta, tb;
            up2(mul2(pk2(g1A, g1B), ACC), ta, tb);
            g1A = ta; g1B = tb;
            up2(mul2(pk2(g2A, g2B), ACC), ta, tb);
            g2A = ta; g2B = tb;
          }
        }
        // packed accumulate on (a, b) register pairs (this form avoids ptxas moves)
        asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
            : "+f"(ax[ka]), "+f"(ax[kb]) : "l"(FF.v), "l"(DX.v));
        asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
            : "+f"(ay[ka]), "+f"(ay[kb]) : "l"(FF.v), "l"(DY.v));
        asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%0, %1};\n\tfma.rn.f32x2 t, %2, %3, t;\n\tmov.b64 {%0, %1}, t;\n\t}"
            : "+f"(az[ka]), "+f"(az[kb]) : "l"(FF.v), "l"(DZ.v));
        if (QUAD) {
          const F2 G1 = pk2(g1A, g1B), G2 = pk2(g2A, g2B);
          F2 AX = pk2(ax[ka], ax[kb]), AY = pk2(ay[ka], ay[kb]), AZ = pk2(az[ka], az[kb]);
          AX = fma2(G2, DX, fma2(G1, QX, AX));
          AY = fma2(G2, DY, fma2(G1, QY, AY));
          AZ = fma2(G2, DZ, fma2(G1, QZ, AZ));
          up2(AX, ax[ka], ax[kb]);
          up2(AY, ay[ka], ay[kb]);
          up2(AZ, az[ka], az[kb]);
        }
      }
      // a target opened cc iff it was active and its res stayed <= cc
      if (STATS) {
#pragma unroll
        for (int k = 0; k < TPL; k++) nop[k] += res[k] <= cc ? 1u : 0u;
        sv_rec += cc < Wn ? 1u : 0u;
        sv_leaf += (cc < Wn && au.x == 0xff800000u) ? 1u : 0u;  // T_acc = -inf: a particle record
      }
      uint32_t rmin = res[0];
#pragma unroll
      for (int k = 1; k < TPL; k++) rmin = min(rmin, res[k]);
      const bool opn = rmin <= cc;
      if (GL == 1) {  // a lane's own group: no vote
        c = opn ? cc + 1u : skip;
      } else if (GL == 32) {
        c = __any_sync(full, opn) ? cc + 1u : skip;
      } else {
        c = (__ballot_sync(full, opn) & gmask2) ? cc + 1u : skip;
      }
    }
    const bool live = c < Wn;
    git += live ? 1u : 0u;
    if (++trip == BH_FOLD_TRIPS) {  // warp-uniform
      trip = 0;
      if (FCNT) {  // the fp32 counts (<= 3 x BH_FOLD_TRIPS each) into the integer ones
#pragma unroll
        for (int j = 0; j < NP; j++) {
          float ca, cb;
          up2(CNT[j], ca, cb);
          if constexpr (FM == 3) {
            s_cnt[2 * j][threadIdx.x] += __float2uint_rn(ca);
            s_cnt[2 * j + 1][threadIdx.x] += __float2uint_rn(cb);
          } else {
            cnt[2 * j] += __float2uint_rn(ca);
            cnt[2 * j + 1] += __float2uint_rn(cb);
          }
          CNT[j] = pk2(0.f, 0.f);
        }
      }
      if constexpr (FM != 0) {
#pragma unroll
        for (int k = 0; k < TPL; k++) {
          if constexpr (FM == 3) {
            s_out[3 * k][threadIdx.x] += ax[k];
            s_out[3 * k + 1][threadIdx.x] += ay[k];
            s_out[3 * k + 2][threadIdx.x] += az[k];
          } else {
            ox[k] += (FoldT)ax[k];
            oy[k] += (FoldT)ay[k];
            oz[k] += (FoldT)az[k];
          }
          ax[k] = ay[k] = az[k] = 0.f;
        }
      }
    }
    if (!__any_sync(full, live)) break;
  }
  asm volatile("" ::: "memory");  // re-read the targets below rather than keep them live in the loop
  Target T[TPL];
  bool v[TPL], own[TPL];
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    const int64_t t = tbase + (int64_t)k * GL;
    v[k] = gin && t < P.n_targets;
    if (v[k]) T[k] = load_target(P, t);
    else { T[k].p = 0; T[k].Li = 0; T[k].s = 0; T[k].me = make_float4(0.f, 0.f, 0.f, 0.f); }
    own[k] = v[k] && (!P.own_check || (T[k].s >= P.own_lo && T[k].s < P.own_hi));
  }
  if (FCNT) {
#pragma unroll
    for (int j = 0; j < NP; j++) {
      float ca, cb;
      up2(CNT[j], ca, cb);
      cnt[2 * j] += __float2uint_rn(ca);
      cnt[2 * j + 1] += __float2uint_rn(cb);
      if constexpr (FM == 3) {
        cnt[2 * j] += s_cnt[2 * j][threadIdx.x];
        cnt[2 * j + 1] += s_cnt[2 * j + 1][threadIdx.x];
      }
    }
  }
  double dax[TPL], day[TPL], daz[TPL];
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    if constexpr (FM == 3) {
      dax[k] = (double)s_out[3 * k][threadIdx.x] + (double)ax[k];
      day[k] = (double)s_out[3 * k + 1][threadIdx.x] + (double)ay[k];
      daz[k] = (double)s_out[3 * k + 2][threadIdx.x] + (double)az[k];
    } else if constexpr (FM == 1 || FM == 2) {
      dax[k] = (double)ox[k] + (double)ax[k];
      day[k] = (double)oy[k] + (double)ay[k];
      daz[k] = (double)oz[k] + (double)az[k];
    } else {
      dax[k] = (double)ax[k];
      day[k] = (double)ay[k];
      daz[k] = (double)az[k];
    }
  }
  if (P.gcost) {
#pragma unroll
    for (int k = 0; k < TPL; k++)
      if (v[k]) P.gcost[T[k].s] = git;  // this walk's cost of the target's group
  }
  unsigned long long wc = 0, wo = 0;
  bool redo[TPL];
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    redo[k] = own[k] && res[k] >= BH_DROP;
    if (!CONT && v[k] && res[k] < BH_DROP) cnt[k] -= 1u;  // own record: "accepted", zero contribution
    wc += (own[k] && !redo[k]) ? cnt[k] : 0u;
    if (STATS) wo += own[k] ? nop[k] : 0u;
  }
  for (int o = 16; o; o >>= 1) {
    wc += __shfl_xor_sync(full, wc, o);
    if (STATS) wo += __shfl_xor_sync(full, wo, o);
  }
  if (lane == 0 && wc) {
    atomicAdd(&P.st->interactions, wc);
    atomicAdd(&P.st->interactions_cum, wc);
  }
  if (STATS) {
    unsigned long long r1 = sv_rec, r2 = sv_leaf;
    for (int o = 16; o; o >>= 1) {
      r1 += __shfl_xor_sync(full, r1, o);
      r2 += __shfl_xor_sync(full, r2, o);
    }
    if (lane == 0) {
      if (wo) {
        atomicAdd(&P.st->opens, wo);
        atomicAdd(&P.st->opens_cum, wo);
      }
      atomicAdd(&P.st->iters, r1);
      atomicAdd(&P.st->reserved0, r2);
    }
  }
#pragma unroll
  for (int k = 0; k < TPL; k++) {
    if (!own[k]) continue;
    if (redo[k])
      push_resume(P, tbase + (int64_t)k * GL, res[k], dax[k], day[k], daz[k], cnt[k],
                  (!CONT && T[k].Li < (res[k] & ~BH_DROP)) ? 1u : 0u);
    else finish(P, T[k], dax[k], day[k], daz[k], cnt[k]);
  }
}

// world > 1: the P = 1 groups (GT consecutive sorted positions) that hold at
// least one particle of this rank's storage range [lo, hi)
__global__ void k_own_group_flags(const uint32_t *__restrict__ vals, uint32_t *__restrict__ flag, int64_t n, int gt,
                                  uint32_t lo, uint32_t hi) {
  const int64_t ng = (n + gt - 1) / gt;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g < ng) {
    uint32_t f = 0;
    const int64_t e = (g + 1) * gt < n ? (g + 1) * gt : n;
    for (int64_t t = g * gt; t < e; t++) {
      const uint32_t s = vals[t];
      f |= (s >= lo && s < hi) ? 1u : 0u;
    }
    flag[g] = f;
  }
  if (g == ng) flag[ng] = 0;
}
__global__ void k_own_group_compact(const uint32_t *__restrict__ pre, uint32_t *__restrict__ list, int64_t ng,
                                    uint32_t *__restrict__ count) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g < ng && pre[g + 1] != pre[g]) list[pre[g]] = (uint32_t)g;
  if (g == ng) *count = pre[ng];
}

// walk_group code -> lanes per group and targets per lane (66 / 67 / 68: 8 /
// 4 / 2 lanes x 2 targets; 69 / 70: 2 / 1 lanes x 4 targets)
int walk_lanes(int group) { return group == 66 ? 8 : group == 68 || group == 69 ? 2 : group == 70 ? 1 : 4; }
static int walk_tpl(int group) { return group == 69 || group == 70 ? 4 : 2; }

cudaError_t launch_walk(const Workspace &W, const WalkArgs &a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  WalkParams P;
  P.rec = W.rec;
  P.quad = a.quad && W.qrec;
  P.qrec = P.quad ? W.qrec : nullptr;
  P.lvl_mom = W.lvl_mom;
  P.rec_item = W.rec_item;
  P.nstart = W.nstart;
  P.vals = W.vals[a.buf];
  P.uid = W.uid;
  P.st = W.status;
  P.icount = W.icount;
  P.redo = W.redo;
  P.gcost = !getenv("BH_NO_GROUP_ORDER") ? W.gcost : nullptr;
  P.resume = W.resume;
  P.cap_resume = W.cap_resume;
  P.resume_stack = W.resume_stack > 0 && W.resume_stack < RESUME_STACK ? W.resume_stack : RESUME_STACK;
  P.need_cont = a.need_cont;
  P.pos4 = W.pos4;
  P.vel4 = W.vel4;
  P.acc_out = a.acc_out;
  P.user_order = a.user_order;
  P.n_targets = a.n;
  P.mode = a.mode;
  P.eps2 = a.eps2;
  P.G = a.G;
  P.kick = a.kick;
  P.dt = a.dt;
  P.theta2 = a.theta2;
  P.own_lo = a.own_lo;
  P.own_hi = a.own_hi;
  P.own_check = a.own_check;
  P.num_sms = a.num_sms > 0 ? a.num_sms : 148;
  P.n_peers = a.mode == 1 ? a.n_peers : 0;
  for (int k = 0; k < BH_MAX_PEERS; k++) P.peer_pos4[k] = k < P.n_peers ? a.peer_pos4[k] : nullptr;
  const int GL = walk_lanes(a.group), GT = walk_tpl(a.group) * GL;
  const int64_t ng_all = (a.n + GT - 1) / GT;
  int64_t ng_max = ng_all;
  P.group_list = nullptr;
  P.n_groups_dev = nullptr;
  if (a.own_check) {
    // the list of P = 1 groups with an own particle (in W.targets) and its
    // length on the device; flags and scan in accu (ng + 1 u32 fit in 3 n floats)
    uint32_t *flag = (uint32_t *)W.accu;
    const unsigned gb = (unsigned)((ng_all + 1 + 255) / 256);
    k_own_group_flags<<<gb, 256, 0, s>>>(P.vals, flag, a.n, GT, a.own_lo, a.own_hi);
    cudaError_t e = launch_scan_u32(flag, ng_all + 1, W.scan_tmp, s);
    if (e != cudaSuccess) return e;
    uint32_t *cnt = &W.status->n_own_groups;
    k_own_group_compact<<<gb, 256, 0, s>>>(flag, W.targets, ng_all, cnt);
    P.group_list = W.targets;
    P.n_groups_dev = cnt;
    const int64_t own_n = (int64_t)a.own_hi - a.own_lo;
    ng_max = own_n < ng_all ? own_n : ng_all;  // every own particle is in one group
  }
  if (ng_max > 0) {
    constexpr int WB = BH_WALK_BLOCK;
    const unsigned grid = (unsigned)((ng_max + WB / GL - 1) / (WB / GL));
    const bool cont = a.need_cont;
#define BH_WALK_LAUNCH(GLv, NPv)                                                      \
  if (a.stats) {                                                                 \
    if (P.quad) {                                                                \
      if (cont) k_walk<GLv, NPv, true, true, true><<<grid, WB, 0, s>>>(P);            \
      else k_walk<GLv, NPv, false, true, true><<<grid, WB, 0, s>>>(P);                \
    } else {                                                                     \
      if (cont) k_walk<GLv, NPv, true, false, true><<<grid, WB, 0, s>>>(P);           \
      else k_walk<GLv, NPv, false, false, true><<<grid, WB, 0, s>>>(P);               \
    }                                                                            \
  } else {                                                                       \
    if (P.quad) {                                                                \
      if (cont) k_walk<GLv, NPv, true, true, false><<<grid, WB, 0, s>>>(P);           \
      else k_walk<GLv, NPv, false, true, false><<<grid, WB, 0, s>>>(P);               \
    } else {                                                                     \
      if (cont) k_walk<GLv, NPv, true, false, false><<<grid, WB, 0, s>>>(P);          \
      else k_walk<GLv, NPv, false, false, false><<<grid, WB, 0, s>>>(P);              \
    }                                                                            \
  }
    switch (a.group) {
      case 66: BH_WALK_LAUNCH(8, 1) break;
      case 68: BH_WALK_LAUNCH(2, 1) break;
      case 69: BH_WALK_LAUNCH(2, 2) break;
      case 70: BH_WALK_LAUNCH(1, 2) break;
      default: BH_WALK_LAUNCH(4, 1) break;
    }
#undef BH_WALK_LAUNCH
  }
  launch_walk_resume(P, a.n, s);
  return cudaGetLastError();
}

}  // namespace bh
