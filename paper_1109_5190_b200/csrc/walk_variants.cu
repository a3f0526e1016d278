// walk_variants.cu -- K6 walk kernels other than the production k_walk2:
// k_walk (one target per lane; group sizes 1..32 and the per-level statistics
// pass) and the k_walk_lane family (walk_group 80..85, 90..95).  Same per-lane
// semantics and fp32 operation sequence as k_walk2 (walk_common.cuh).
#include "walk_common.cuh"

namespace bh {

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

cudaError_t launch_walk_lane(const WalkParams &P, int group, bool cont, int64_t n_targets, cudaStream_t s) {
  // group walk (k_walk_lane): lanes per group x targets per lane
  //   80: 1 x 4   81: 1 x 2   82: 2 x 4   83: 2 x 2   84: 4 x 2   85: 4 x 4
  //   (persistent, SM-local tickets); +10: the same, one group per slot
  const bool persist = group < 90;
  const int code = persist ? group : group - 10;
  cudaError_t e = cudaMemsetAsync(P.st->sm_next, 0, sizeof(P.st->sm_next), s);  // the ticket counters
  if (e != cudaSuccess) return e;
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
  const int64_t ngroups = (n_targets + tpg - 1) / tpg;
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
  return cudaSuccess;
}

void launch_walk_simple(const WalkParams &P, int group, bool stats, int64_t n_targets, cudaStream_t s) {
  const unsigned grid = (unsigned)((n_targets + 255) / 256);
#define BH_WALK_CASE(g)                                                     \
  case g:                                                                   \
    if (stats) k_walk<g, true><<<grid, 256, 0, s>>>(P);                     \
    else k_walk<g, false><<<grid, 256, 0, s>>>(P);                          \
    break;
  switch (group) {
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

}  // namespace bh
