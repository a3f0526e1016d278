// com.cu -- K5: level-synchronous bottom-up mass and centre of mass.
//
// PAPER.md:60-61 (§1): the octree is used "to compute center of mass and force
// on each of the cubes"; Fig. 2 caption: P3 and P4 "may be
// replaced by an equivalent centroid".  Reading L14: M and
// MX = sum m x are fp64 sums over the children in Morton digit order, left to
// right from 0 (bucket members in sorted order); a leaf contributes M = m,
// MX = m x, exact in fp64 (24 x 24-bit products); com = MX / M.  Every fp64
// operation is an explicit round-to-nearest intrinsic, so the result is
// bit-identical to the oracle's recursive sums.
//
// One launch per level l = 21 .. 0 over that level's Morton-ordered items (K4,
// tree.cu): an internal node's children are the contiguous range
// [clo(node), clo(next item)) of the level-(l+1) items, whose fp64 moments the
// previous launch (or K4, for particles: (m, m x)) wrote in level order, so
// the sums stream.  skip() comes bottom-up too (the last child's).  The kernel
// also emits each node's fp32 walk record: com32 = RN(com), M32 = RN(M), and the two fp32 thresholds of the
// force walk's MAC filter (walk.cu):
//   accept for sure  if d2_32 > T_acc,   open for sure  if d2_32 < T_rej,
//   otherwise the walk re-evaluates the exact fp64 test of the oracle.
// With r = s_l / theta the exact test is d > r (s^2 < theta^2 d^2).  The fp32
// distance of the walk differs from the oracle's fp64 distance by at most
//   |d32 - d| <= u d + u(1+u) |c32|   (u = 2^-24: subtraction + com rounding)
// and the fp32 sum of squares (mul, fma, fma) by a relative 3u; delta = 1e-12
// covers the oracle's own fp64 rounding.  Hence (safety factor 1.5 on each term)
//   T_acc = RU(((r(1+delta) + b) / (1-a))^2 (1+g)),
//   T_rej = RD(((r(1-delta) - b) / (1+a))^2 (1-g))   (or -inf if negative),
// with a = 1.5u, b = 1.5u |c32|, g = 4.5u.  theta == 0: T_acc = T_rej = +inf.
// For theta >= 0.57 T_acc is also raised to the bound of the node's bounding
// radius, so the walk needs no containment test (ContFold below, reading R2).
#include <math.h>

#include "bh_internal.cuh"

// BH_EPS_FOLD (bh_internal.cuh, default 1): the filter's thresholds are in the softened
// domain, r2_32 = fma(dz, dz, fma(dy, dy, fma(dx, dx, eps2_32))) against
//   T_acc = RU((A^2 + eps2_32) (1+g)),  T_rej = RD((B^2 + eps2_32) (1-g)),
// so the walk compares the same r2 it feeds to rsqrt (one packed add fewer per
// target pair and record).  The three fma roundings of positive terms keep the
// relative 3u of the unsoftened sum (g unchanged), and d <= r <=> d^2 + eps^2
// <= r^2 + eps^2, so the decisions, hence every result, are those of the exact
// test as before.
#ifndef BH_MOM_COMPACT
// K5: internal nodes queued per warp (k_moments_level); 2 = where the
// per-node work is heavy (the containment fold's radii, quadrupoles): cfg5
// moments 3.25 -> 2.66 ms, while cfg4's light nodes lost (0.603 -> 0.645)
#define BH_MOM_COMPACT 2
#endif
#ifndef BH_TIGHT_COM
#define BH_TIGHT_COM 1
#endif
#ifndef BH_MOM_PREFETCH
#define BH_MOM_PREFETCH 2  // (2 vs 1/3/4: best on cfg4 and on cfg5 with the containment fold)
#endif
#ifndef BH_MOM_WAVES
#define BH_MOM_WAVES 4  // grid cap in blocks per SM: one resident wave at 64 registers (4 vs 8: cfg5 moments 2.684 -> 2.646 ms, cfg3 0.178 -> 0.171, cfg4 0.614 -> 0.611; 3: worse, 2: cfg5 3.44)
#endif
#ifndef BH_MOM_MINB
#define BH_MOM_MINB 4  // 64 registers: 4 blocks (32 warps) per SM (the containment fold needs 66 unbounded: 3 blocks, cfg5 moments +20%)
#endif
// (multipole = 2 kernels unbounded: their quadrupole sums would spill)
#define BH_MOM_BOUNDS __launch_bounds__(256, QUAD ? 1 : BH_MOM_MINB)

namespace bh {

__device__ __forceinline__ float round_up_f(double x) {
  float f = __double2float_ru(x);
  return f;
}
__device__ __forceinline__ float round_down_f(double x) {
  float f = __double2float_rd(x);
  return f;
}

// multipole = 2 (reading L25; the oracle's step 9): m (3 y y^T - |y|^2 I) of a
// point mass at offset y, added to Q (xx yy zz xy xz yz) with the oracle's
// fp64 operation order, so the quadrupoles are bit-identical too
__device__ __forceinline__ void add_point_quad(double Q[6], double m, double y0, double y1, double y2) {
  double r2 = __dmul_rn(y0, y0);
  r2 = __dadd_rn(r2, __dmul_rn(y1, y1));
  r2 = __dadd_rn(r2, __dmul_rn(y2, y2));
  Q[0] = __dadd_rn(Q[0], __dmul_rn(m, __dsub_rn(__dmul_rn(__dmul_rn(3.0, y0), y0), r2)));
  Q[1] = __dadd_rn(Q[1], __dmul_rn(m, __dsub_rn(__dmul_rn(__dmul_rn(3.0, y1), y1), r2)));
  Q[2] = __dadd_rn(Q[2], __dmul_rn(m, __dsub_rn(__dmul_rn(__dmul_rn(3.0, y2), y2), r2)));
  Q[3] = __dadd_rn(Q[3], __dmul_rn(m, __dmul_rn(__dmul_rn(3.0, y0), y1)));
  Q[4] = __dadd_rn(Q[4], __dmul_rn(m, __dmul_rn(__dmul_rn(3.0, y0), y2)));
  Q[5] = __dadd_rn(Q[5], __dmul_rn(m, __dmul_rn(__dmul_rn(3.0, y1), y2)));
}

// Containment folded into the fp32 filter (theta >= 0.57 with eps > 0, so the
// fast walk needs no per-visit containment test).  Every item carries a
// bounding radius R about its com: R(particle) = 0, R(node) >= max over
// children of |com - com_child| + R_child (child coms from their fp64 moments,
// with a reciprocal instead of a division and the rounding added), so every
// particle of the node lies within R of its com, and a target inside the node
// (one of its particles) is at distance <= R.  T_acc is raised to the
// bound of R (the T_acc error model with r -> R): a node that may contain the
// target is then never accepted for sure, and the band between T_rej and that
// bound goes to the exact re-walk, which tests containment (reading L5).  For
// most nodes R < s/theta already and nothing changes.
struct ContFold {
  float *lvl_rad;
  int on;
};

// one internal node of level `level` at item t (record c, children [lo, hi) of the next level)
template <bool QUAD, bool FOLD>
__device__ __forceinline__ void moments_node(int level, uint32_t t, uint32_t c, uint32_t lo, uint32_t hi, uint32_t off,
                                             uint32_t off1, double r_lvl, double theta, double eps2d,
                                             const uint32_t *__restrict__ item_rec, uint32_t *__restrict__ lvl_skip,
                                             double4 *__restrict__ lvl_mom, Rec *__restrict__ rec,
                                             double *__restrict__ lvl_q,
                                             double *__restrict__ qmom, float4 *__restrict__ qrec,
                                             const ContFold cf, const DevStatus *__restrict__ st) {
  const uint32_t skip = lvl_skip[off1 + hi - 1];  // the last child's
  // the children in digit order (reading L14): a particle contributes
  // (m, m x), an internal node its (M, MX); the first BH_MOM_PREFETCH are
  // loaded at once
  double4 q[BH_MOM_PREFETCH];
#pragma unroll
  for (int k = 0; k < BH_MOM_PREFETCH; k++)
    q[k] = lo + k < hi ? lvl_mom[off1 + lo + k] : make_double4(0.0, 0.0, 0.0, 0.0);
  double M = 0.0, X = 0.0, Y = 0.0, Z = 0.0;
#pragma unroll
  for (int k = 0; k < BH_MOM_PREFETCH; k++) {
    if (lo + k < hi) {
      M = __dadd_rn(M, q[k].x);
      X = __dadd_rn(X, q[k].y);
      Y = __dadd_rn(Y, q[k].z);
      Z = __dadd_rn(Z, q[k].w);
    }
  }
  for (uint32_t j = lo + BH_MOM_PREFETCH; j < hi; j++) {
    const double4 r = lvl_mom[off1 + j];
    M = __dadd_rn(M, r.x);
    X = __dadd_rn(X, r.y);
    Y = __dadd_rn(Y, r.z);
    Z = __dadd_rn(Z, r.w);
  }
  lvl_mom[off + t] = make_double4(M, X, Y, Z);
  lvl_skip[off + t] = skip;
  // com = MX / M: the exact quotients where the quadrupoles need them (they are
  // compared bit for bit with the oracle's); else one reciprocal (<= 1.5 ulp
  // of fp64 off, far inside the fp32 filter's com-rounding term)
  double cx, cy, cz;
  if (QUAD) {
    cx = __ddiv_rn(X, M); cy = __ddiv_rn(Y, M); cz = __ddiv_rn(Z, M);
  } else {
    const double iM = 1.0 / M;
    cx = X * iM; cy = Y * iM; cz = Z * iM;
  }
  // a massless node has no com (0/0, as in the oracle): its record gets a finite
  // dummy point and thresholds that always open it, so nothing NaN reaches the
  // walk's branch-free arithmetic (0 x NaN)
  const bool massless = !(M > 0.0);
  const float fx = massless ? 0.f : __double2float_rn(cx), fy = massless ? 0.f : __double2float_rn(cy),
              fz = massless ? 0.f : __double2float_rn(cz);
  double Rn = 0.0;
  if (FOLD) {
    const double cn = fabs(cx) + fabs(cy) + fabs(cz);
    // one child's reach |com - com_j| + R_j (+ rounding); a massless child: a
    // particle's position from its record, a massless node unbounded
    auto reach = [&](const double4 mj, float rj, uint32_t j) -> double {
      if (mj.x > 1e-30) {
        // |com - com_j| = |M_j com - MX_j| / M_j: the difference in fp64 (one
        // fma per axis, no cancellation loss), then fp32.  Error budget of d
        // (relative, u = 2^-24): 3 conversions to fp32 (3u, on the squares 6u),
        // the sum of squares (3u), rsqrtf (<= 2 ulp), q2 * rsqrt (u), the
        // conversion of M_j (u) and its approximate reciprocal (<= 2 ulp), the
        // last multiply (u): ~18u = 1.1e-6, covered by the factor (1 + 1.5e-6).
        // An overflow of the fp32 difference (large masses: q2 = +inf, rsqrt 0,
        // inf * 0 = NaN) or of d takes the fp64 route below instead -- a NaN
        // must never reach the max over children.
        const float e0 = (float)fma(mj.x, cx, -mj.y), e1 = (float)fma(mj.x, cy, -mj.z),
                    e2 = (float)fma(mj.x, cz, -mj.w);
        const float q2 = fmaf(e2, e2, fmaf(e1, e1, e0 * e0));
        const float d = q2 > 0.f ? q2 * rsqrtf(q2) * __fdividef(1.0f, (float)mj.x) : 0.f;
        if (d < INFINITY) return (double)d * (1.0 + 1.5e-6) + (double)rj;
      }
      double px, py, pz;
      if (mj.x > 0.0) {  // (tiny masses, or an fp32 overflow: the slow exact route)
        px = mj.y / mj.x;
        py = mj.z / mj.x;
        pz = mj.w / mj.x;
      } else {  // massless: a particle's position from its record; a node unbounded
        const uint32_t ec = item_rec[off1 + j];
        if (!(ec & ITEM_LEAF)) return INFINITY;
        const float4 pp = rec[ec & ~ITEM_LEAF].cm;
        px = pp.x;
        py = pp.y;
        pz = pp.z;
      }
      const double ex = cx - px, ey = cy - py, ez = cz - pz;
      const double d = sqrt(ex * ex + ey * ey + ez * ez);
      return d + (double)rj + 1e-14 * (cn + fabs(px) + fabs(py) + fabs(pz) + d);
    };
    // the children again (just read for the sums: cached)
    // (NaN-propagating max: fmax would drop a NaN reach)
    for (uint32_t j = lo; j < hi; j++) {
      const double rj = reach(lvl_mom[off1 + j], cf.lvl_rad[off1 + j], j);
      Rn = (rj > Rn || rj != rj) ? rj : Rn;
    }
    if (!(Rn <= 1e300)) Rn = INFINITY;  // (also a NaN com of a massless node)
    cf.lvl_rad[off + t] = Rn == INFINITY ? INFINITY : round_up_f(Rn * (1.0 + 1e-12));
  }
  if (QUAD) {
    // the quadrupole about (cx, cy, cz): the children in digit order, each its
    // own Q plus its mass at its com's offset (parallel-axis rule)
    double Q[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (uint32_t j = lo; j < hi; j++) {
      const uint32_t ec = item_rec[off1 + j];
      if (ec & ITEM_LEAF) {
        const float4 pp = rec[ec & ~ITEM_LEAF].cm;
        add_point_quad(Q, (double)pp.w, __dsub_rn((double)pp.x, cx), __dsub_rn((double)pp.y, cy),
                       __dsub_rn((double)pp.z, cz));
      } else {
        const double *qc = lvl_q + 6 * (size_t)(off1 + j);
#pragma unroll
        for (int k = 0; k < 6; k++) Q[k] = __dadd_rn(Q[k], qc[k]);
        const double4 mc = lvl_mom[off1 + j];
        add_point_quad(Q, mc.x, __dsub_rn(__ddiv_rn(mc.y, mc.x), cx), __dsub_rn(__ddiv_rn(mc.z, mc.x), cy),
                       __dsub_rn(__ddiv_rn(mc.w, mc.x), cz));
      }
    }
#pragma unroll
    for (int k = 0; k < 6; k++) {
      qmom[6 * (size_t)c + k] = Q[k];
      lvl_q[6 * (size_t)(off + t) + k] = Q[k];
    }
    // the walk's copy is -Q in fp32 (walk.cu: the minus sign of the field's
    // first term rides on Q, exactly)
    if (massless) {
      qrec[2 * (size_t)c] = make_float4(0.f, 0.f, 0.f, 0.f);
      qrec[2 * (size_t)c + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      qrec[2 * (size_t)c] = make_float4(-__double2float_rn(Q[0]), -__double2float_rn(Q[1]),
                                        -__double2float_rn(Q[2]), -__double2float_rn(Q[3]));
      qrec[2 * (size_t)c + 1] = make_float4(-__double2float_rn(Q[4]), -__double2float_rn(Q[5]), 0.f, 0.f);
    }
  }
  float tacc, trej;
  // the filter's constants: u = 2^-24; 1 / (1 -+ a) as products (their
  // rounding, a few fp64 ulp, sits inside the 4e-15 slack)
  constexpr double u = 5.9604644775390625e-08;
  constexpr double a = 1.5 * u, g = 4.5 * u, delta = 1e-12;
  constexpr double i1ma = 1.0 / (1.0 - a), i1pa = 1.0 / (1.0 + a);
  double C = 0.0;
  if (!(theta > 0.0) || massless) {
    tacc = INFINITY;
    trej = INFINITY;
  } else {
    const double r = r_lvl;  // s_l / theta of this level (the kernel's)
    C = sqrt((double)fx * fx + (double)fy * fy + (double)fz * fz);
    // first-order bounds (u: com rounding |c32 - c64| <= u(1+u)|c32|, one
    // rounding of the subtraction, <= 3 roundings in the fp32 sum of squares)
    // with a safety factor 1.5 on every term.  BH_TIGHT_COM: the com term is
    // the node's actual rounding displacement |c32 - c64| instead of its
    // bound (c32 - c64 is exact in fp64; its norm is padded by 1e-6 relative,
    // and 1e-15 |c| covers c64's reciprocal against the oracle's quotient,
    // <= 2.5 fp64 ulp per axis) -- on average ~3x narrower, and it dominates
    // the band wherever r << |c| (cfg5: 100x the subtraction term at level 10)
#if BH_TIGHT_COM
    const double ex = (double)fx - cx, ey = (double)fy - cy, ez = (double)fz - cz;
    const double b = sqrt(ex * ex + ey * ey + ez * ez) * (1.0 + 1e-6) + 1e-15 * C;
#else
    const double b = 1.5 * u * C;
#endif
    const double A = (r * (1.0 + delta) + b) * i1ma;
    tacc = round_up_f((A * A + eps2d) * (1.0 + g) * (1.0 + 4e-15));
    const double B = (r * (1.0 - delta) - b) * i1pa;
    trej = B > 0.0 ? round_down_f((B * B + eps2d) * (1.0 - g) * (1.0 - 4e-15)) : -INFINITY;
    // Levels 20-21: fp32 quantisation can place a particle up to 0.19 grid
    // quanta outside its key-space cell, so there (and only there) a cell
    // containing the target could pass s/d < theta for theta < 1/sqrt(3).
    // The fast walk skips the containment test (walk.cu); never accepting
    // these cells in the fp32 filter routes every such decision to the exact
    // re-walk, which tests containment.
    if (level >= 20) tacc = INFINITY;
    if (FOLD && level < 20) {
      const double A = (Rn * (1.0 + 1e-12) + b) * i1ma;
      tacc = Rn == INFINITY ? INFINITY : fmaxf(tacc, round_up_f((A * A + eps2d) * (1.0 + g) * (1.0 + 4e-15)));
    }
  }
  Rec r;
  r.cm = make_float4(fx, fy, fz, __double2float_rn(M));
  r.aux = make_uint4(__float_as_uint(tacc), __float_as_uint(trej), skip, BH_DROP | c);  // drop word (walk.cu)
  rec[c] = r;
}

// one launch per level over the level's items (a node after its children).
// (Measured alternative, not kept: one chunk-local pass over the nodes inside
// 4096-particle chunks plus per-level launches over the boundary nodes -- cfg4
// 0.83 vs 0.64 ms, cfg5 4.05 vs 3.56 ms: the per-chunk level loop is latency
// bound, profiles/r2_summary.md.)
template <bool QUAD, bool FOLD>
__global__ void BH_MOM_BOUNDS k_moments_level(int level, const DevStatus *__restrict__ st,
                                                       const uint32_t *__restrict__ item_rec,
                                                       const uint32_t *__restrict__ item_clo,
                                                       uint32_t *__restrict__ lvl_skip,
                                                       double4 *__restrict__ lvl_mom, Rec *__restrict__ rec,
                                                       double theta, double eps2d,
                                                       double *__restrict__ lvl_q, double *__restrict__ qmom,
                                                       float4 *__restrict__ qrec, const ContFold cf) {
  if (st->err & ERR_NODE_OVERFLOW) return;
  const uint32_t cnt = st->lvl_count[level];
  const uint32_t off = st->lvl_offset[level];
  const uint32_t cnt1 = st->lvl_count[level + 1];
  const uint32_t off1 = st->lvl_offset[level + 1];
  const double r_lvl = ldexp((double)st->L, -level) / theta;  // s_l / theta
  constexpr bool COMPACT = BH_MOM_COMPACT == 1 || (BH_MOM_COMPACT == 2 && (FOLD || QUAD));
  if constexpr (COMPACT) {
  // Warp compaction: most items of a level are particles (K4 finished them),
  // so a lane per item leaves ~2/3 of the lanes idle in moments_node.  Each
  // warp scans windows of 32 items (one coalesced load), queues the internal
  // nodes in shared memory in item order (ballot ranks) and runs
  // moments_node 32 queued nodes at a time with every lane busy.
  __shared__ uint32_t s_qt[256 / 32][64], s_qe[256 / 32][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  uint32_t *qt = s_qt[w], *qe = s_qe[w];
  uint32_t qn = 0;  // warp-uniform
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  auto run = [&](uint32_t tq, uint32_t eq) {
    const uint32_t lq = item_clo[off + tq];
    const uint32_t hq = tq + 1 < cnt ? item_clo[off + tq + 1] : cnt1;
    moments_node<QUAD, FOLD>(level, tq, eq, lq, hq, off, off1, r_lvl, theta, eps2d, item_rec, lvl_skip, lvl_mom, rec,
                             lvl_q, qmom, qrec, cf, st);
  };
  for (uint32_t wb = (blockIdx.x * (blockDim.x >> 5) + w) * 32u; wb < cnt; wb += nwarps * 32u) {
    const uint32_t tw = wb + lane;
    const uint32_t ew = tw < cnt ? item_rec[off + tw] : ITEM_LEAF;
    const bool in = !(ew & ITEM_LEAF);
    const uint32_t bal = __ballot_sync(0xffffffffu, in);
    if (in) {
      const uint32_t pos = qn + __popc(bal & lt);
      qt[pos] = tw;
      qe[pos] = ew;
    }
    qn += __popc(bal);
    __syncwarp();
    if (qn >= 32u) {
      const uint32_t tq = qt[lane], eq = qe[lane];
      __syncwarp();
      if ((uint32_t)lane < qn - 32u) {
        qt[lane] = qt[lane + 32];
        qe[lane] = qe[lane + 32];
      }
      qn -= 32u;
      __syncwarp();
      run(tq, eq);
    }
  }
  if ((uint32_t)lane < qn) run(qt[lane], qe[lane]);
  } else {
  // one round trip for an item, one for its children (loads hoisted so they
  // are in flight together); the next item's loads are issued before this
  // one's children are summed
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t e = ITEM_LEAF, lo = 0, hi = 0;
  if (t < cnt) {
    e = item_rec[off + t];
    lo = item_clo[off + t];
    hi = t + 1 < cnt ? item_clo[off + t + 1] : cnt1;
  }
  for (; t < cnt; t += stride) {
    const uint32_t tn = t + stride;
    uint32_t en = ITEM_LEAF, lon = 0, hin = 0;
    if (tn < cnt) {
      en = item_rec[off + tn];
      lon = item_clo[off + tn];
      hin = tn + 1 < cnt ? item_clo[off + tn + 1] : cnt1;
    }
    const uint32_t ecur = e, locur = lo, hicur = hi;
    e = en;
    lo = lon;
    hi = hin;
    if (ecur & ITEM_LEAF) continue;  // a particle: K4 wrote its record and moments
    moments_node<QUAD, FOLD>(level, t, ecur, locur, hicur, off, off1, r_lvl, theta, eps2d, item_rec, lvl_skip, lvl_mom, rec,
                       lvl_q, qmom, qrec, cf, st);
  }
  }
}


cudaError_t launch_moments(const Workspace &W, int64_t n, double theta, float eps2, int cont_fold, cudaStream_t s,
                           int *launches) {
  ContFold cf;
  cf.lvl_rad = W.lvl_rad;
  cf.on = cont_fold;
  if (n < 2) return cudaSuccess;
  const double eps2d = BH_EPS_FOLD ? (double)eps2 : 0.0;  // the walk's fp32 eps^2, exactly
  // grid: enough blocks for the widest level (at most n items), capped at
  // BH_MOM_WAVES blocks per SM (one resident wave; the items are grid-strided)
  int64_t need = (n + 255) / 256;
  int64_t lim = 148 * BH_MOM_WAVES;
  int grid = (int)(need < lim ? need : lim);
  if (grid < 1) grid = 1;
  for (int l = BH_MAXLEVEL; l >= 0; l--) {
#define BH_MOM_LAUNCH(Q, F)                                                                                  \
  k_moments_level<Q, F><<<grid, 256, 0, s>>>(l, W.status, W.item_rec, W.item_clo, W.lvl_skip, W.lvl_mom, W.rec, \
                                             theta, eps2d, W.lvl_q, W.qmom, W.qrec, cf)
    if (W.qmom) {
      if (cf.on) BH_MOM_LAUNCH(true, true);
      else BH_MOM_LAUNCH(true, false);
    } else {
      if (cf.on) BH_MOM_LAUNCH(false, true);
      else BH_MOM_LAUNCH(false, false);
    }
#undef BH_MOM_LAUNCH
    if (launches) (*launches)++;
  }
  return cudaGetLastError();
}

}  // namespace bh
