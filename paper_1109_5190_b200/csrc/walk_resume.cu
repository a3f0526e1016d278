// walk_resume.cu -- K6 continuation: targets whose fp32 MAC test was
// inconclusive finish their walk here with the oracle's fp64 test.
#include "walk_common.cuh"

namespace bh {

__device__ __noinline__ bool exact_accept(const double4 *__restrict__ lvl_mom, const uint32_t *__restrict__ rec_item, uint32_t c, uint32_t level, float x,
                                          float y, float z, double L, double theta2) {
  // the oracle's fp64 test (DESIGN.md §3 L4), operation for operation
  double4 m = lvl_mom[rec_item[c]];
  double cx = __ddiv_rn(m.y, m.x), cy = __ddiv_rn(m.z, m.x), cz = __ddiv_rn(m.w, m.x);
  double dx = __dsub_rn(cx, (double)x), dy = __dsub_rn(cy, (double)y), dz = __dsub_rn(cz, (double)z);
  double d2 = __dmul_rn(dx, dx);
  d2 = __dadd_rn(d2, __dmul_rn(dy, dy));
  d2 = __dadd_rn(d2, __dmul_rn(dz, dz));
  double s = ldexp(L, -(int)level);
  double s2 = __dmul_rn(s, s);
  return s2 < __dmul_rn(theta2, d2);
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
#if BH_EPS_FOLD
  const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmaf_rn(dx, dx, P.eps2)));  // softened (com.cu)
  const float r2 = d2;
#else
  const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
  const float r2 = __fadd_rn(d2, P.eps2);
#endif
  const bool cont = (c <= T.Li) & (au.z > T.Li);
  bool acc = !cont & (d2 > __uint_as_float(au.x));
  if (!cont && !acc && d2 >= __uint_as_float(au.y)) {
    acc = exact_accept(P.lvl_mom, P.rec_item, c, record_level(P, c), T.me.x, T.me.y, T.me.z, Ld, P.theta2);
    A.fb++;
  }
  if (acc) {
    const float inv = rsqrt_fast(r2);
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
    double pax = 0.0, pay = 0.0, paz = 0.0;
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
      finish(P, T, pax + A.ax, pay + A.ay, paz + A.az, cnt);
    }
    __syncwarp();
  }
}

// a fixed grid, grid-stride over the device-side queue (lanes dense in queue order)
void launch_walk_resume(const WalkParams &P, int64_t n_targets, cudaStream_t s) {
  int64_t eg = (n_targets + RESUME_WARPS - 1) / RESUME_WARPS;
  if (eg > 148 * 16) eg = 148 * 16;
  k_walk_resume<<<(unsigned)eg, 32 * RESUME_WARPS, 0, s>>>(P);
}

}  // namespace bh
