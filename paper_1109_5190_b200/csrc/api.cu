// api.cu -- the C ABI of libbh.so (include/bh.h): ctx, workspace carving,
// state load / store, the step driver and the NCCL exchange (K8).
//
// The step driver enqueues, per time step ("a global barrier
// at the tree construction stage of every iteration" = stream order here):
//   K0 bbox -> K1 keys (+ sort histograms) -> K2 8 Onesweep passes (+ tie
//   fix-up) -> K4 LCP / record counts / scan / emit -> K5 22 level passes ->
//   [world > 1: owned-target compaction] -> K6+K7 walk + leapfrog ->
//   [world > 1: K8 grouped ncclBroadcast of every rank's slice of pos4].
#include <float.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "bh_internal.cuh"

using namespace bh;

struct ProfPair {
  cudaEvent_t a, b;
  int phase;
  int launches;
};

struct bh_ctx {
  bh_params p;
  Layout lay;
  Workspace W;
  cudaStream_t stream;
  bool own_stream;
  int64_t own_lo, own_hi;
  std::vector<int64_t> bounds;  // ownership: rank r owns storage ids [bounds[r], bounds[r+1])
  int64_t steps;
  bool tree_valid;
  bool walked;
  int walk_stats;
  int use_graphs;
  cudaGraphExec_t step_graph[3];  // [0]: half kick (first step), [1]: full kick, [2]: bh_advance's first step
  int num_sms;
  int sort_buf;
  int near_sort;        // 1: try the near-sorted path each build (nearsort.cu)
  int cont_fold;        // containment folded into T_acc (com.cu): the walk skips its per-visit test
  // fused exchange (bh_set_peers): the other ranks' pos4 replicas, written by K7
  std::vector<float4 *> peers;
  DevStatus *hstatus;  // pinned
  cudaEvent_t status_ev;
  // bh_advance: the velocity upload runs on io_stream beside the first build
  cudaStream_t io_stream;
  cudaEvent_t io_ev_pos, io_ev_vel;
  bool vel_pending;      // vel4 still to be loaded from vel_src before the next walk
  const float *vel_src;  // device copy of the user-order velocities (null: zero)
  bool status_pending;
  char err[512];
  // profiling
  bool prof;
  std::vector<ProfPair> pending;
  std::vector<cudaEvent_t> free_events;
  double prof_ms[BH_NPHASE];
  int64_t prof_launches[BH_NPHASE];
  int64_t prof_calls;
};

static bh_status fail(bh_ctx *c, bh_status st, const char *fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof c->err, fmt, ap);
    va_end(ap);
  }
  return st;
}

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(ctx, BH_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                      \
  } while (0)

// ---------------------------------------------------------------- layout
namespace bh {

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

Layout make_layout(int64_t n, int world, int64_t node_capacity, int multipole) {
  Layout L;
  memset(&L, 0, sizeof L);
  L.n = n;
  int64_t def_int = n;
  int64_t worst = 21 * n;
  if (worst > ((int64_t)1 << 22)) worst = (int64_t)1 << 22;
  if (worst > def_int) def_int = worst;
  L.cap_rec = node_capacity > 0 ? node_capacity : n + def_int + 64;
  if (L.cap_rec > BH_MAX_RECORDS) L.cap_rec = BH_MAX_RECORDS;  // record indices stay below the walk's drop flag
  L.cap_int = L.cap_rec - n;
  L.cap_resume = n / 8 > 65536 ? n / 8 : 65536;
  if (L.cap_resume > n) L.cap_resume = n;
  // velocities of the own slice; room for 2x the even share so that
  // bh_set_partition can move the boundaries (equal-cost splits)
  L.n_own_max = 2 * ((n + world - 1) / world) + 1;
  if (L.n_own_max > n) L.n_own_max = n;
  L.sort_tiles = (n + SORT_TILE - 1) / SORT_TILE;
  L.scan_tiles = (n + 1 + SCAN_TILE - 1) / SCAN_TILE + 1;
  L.blocks = (n + 1 + 255) / 256;  // tree.cu's particle blocks
  size_t sz[31] = {
      sizeof(DevStatus),                       // 0 status
      (size_t)n * 16,                          // 1 pos4
      (size_t)L.n_own_max * 16,                // 2 vel4
      (size_t)n * 4,                           // 3 uid
      (size_t)n * 8,                           // 4 keys0
      (size_t)n * 8,                           // 5 keys1
      (size_t)n * 4,                           // 6 vals0
      (size_t)n * 4,                           // 7 vals1
      (size_t)n,                               // 8 lcp
      (size_t)(n + 1) * 4,                     // 9 nstart
      (size_t)n * 4,                           // 10 icount
      (size_t)n * 12,                          // 11 accu
      (size_t)(n + 1) * 4,                     // 12 targets
      (size_t)L.scan_tiles * 4,                // 13 scan_tmp
      sizeof(uint32_t) * (SORT_PASSES * SORT_RADIX + 8 + (size_t)SORT_PASSES * L.sort_tiles * SORT_RADIX),  // 14
      sizeof(float) * 8 * BBOX_BLOCKS,         // 15 bbox partials
      (size_t)L.cap_rec * 32,                  // 16 rec (cm + aux)
      (size_t)L.cap_resume * sizeof(ResumeState),  // 17 walk resume states
      (size_t)L.cap_rec * 4,                   // 18 rec_item: level-item index of each record
      (size_t)n * 12,                          // 19 bh_advance: user-order velocities in flight
      (size_t)L.cap_rec * 4,                   // 20 item_rec (level-ordered items)
      (size_t)n * 4,                           // 21 redo list
      (size_t)n * 4,                           // 22 walk cost per particle (its group's trips)
      multipole == 2 ? (size_t)L.cap_rec * 48 : 0,  // 23 quadrupoles fp64 (multipole = 2)
      multipole == 2 ? (size_t)L.cap_rec * 32 : 0,  // 24 quadrupoles fp32 for the walk
      (size_t)L.cap_rec * 4,                   // 25 item_clo
      (size_t)L.cap_rec * 4,                   // 26 lvl_skip
      (size_t)L.cap_rec * 32,                  // 27 lvl_mom
      multipole == 2 ? (size_t)L.cap_rec * 48 : 0,  // 28 lvl_q
      (size_t)BH_NLEVELS * (L.blocks + (L.blocks + 1023) / 1024) * 4,  // 29 blkcnt + segment sums (tree.cu)
      (size_t)L.cap_rec * 4,                   // 30 lvl_rad: bounding radius of each item (containment fold)
  };
  size_t off = 0;
  for (int i = 0; i < 31; i++) {
    L.off[i] = off;
    off += align_up(sz[i]);
  }
  L.total = off;
  return L;
}

void bind_workspace(const Layout &L, void *base, Workspace &W) {
  char *b = (char *)base;
  W.status = (DevStatus *)(b + L.off[0]);
  W.pos4 = (float4 *)(b + L.off[1]);
  W.vel4 = (float4 *)(b + L.off[2]);
  W.uid = (uint32_t *)(b + L.off[3]);
  W.keys[0] = (unsigned long long *)(b + L.off[4]);
  W.keys[1] = (unsigned long long *)(b + L.off[5]);
  W.vals[0] = (uint32_t *)(b + L.off[6]);
  W.vals[1] = (uint32_t *)(b + L.off[7]);
  W.lcp = (uint8_t *)(b + L.off[8]);
  W.nstart = (uint32_t *)(b + L.off[9]);
  W.icount = (uint32_t *)(b + L.off[10]);
  W.accu = (float *)(b + L.off[11]);
  W.targets = (uint32_t *)(b + L.off[12]);
  W.scan_tmp = (uint32_t *)(b + L.off[13]);
  W.sort_hist = (uint32_t *)(b + L.off[14]);
  W.sort_tilectr = W.sort_hist + SORT_PASSES * SORT_RADIX;
  W.sort_status = W.sort_tilectr + 8;
  W.bbox_part = (float *)(b + L.off[15]);
  W.rec = (Rec *)(b + L.off[16]);
  W.resume = (ResumeState *)(b + L.off[17]);
  W.cap_resume = L.cap_resume;
  W.rec_item = (uint32_t *)(b + L.off[18]);
  W.vstage = (float *)(b + L.off[19]);
  W.item_rec = (uint32_t *)(b + L.off[20]);
  W.item_clo = (uint32_t *)(b + L.off[25]);
  W.lvl_skip = (uint32_t *)(b + L.off[26]);
  W.lvl_mom = (double4 *)(b + L.off[27]);
  W.lvl_q = L.off[28] != L.off[29] ? (double *)(b + L.off[28]) : nullptr;
  W.blkcnt = (uint32_t *)(b + L.off[29]);
  W.lvl_rad = (float *)(b + L.off[30]);
  W.redo = (uint32_t *)(b + L.off[21]);
  W.gcost = (uint32_t *)(b + L.off[22]);
  W.qmom = L.off[23] != L.off[24] ? (double *)(b + L.off[23]) : nullptr;
  W.qrec = L.off[24] != L.off[25] ? (float4 *)(b + L.off[24]) : nullptr;
}

// ---------------------------------------------------------------- small kernels
__global__ void k_pack(float4 *__restrict__ pos4, const float *__restrict__ pos, const float *__restrict__ mass,
                       int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) pos4[i] = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], mass[i]);
}

__global__ void k_iota(uint32_t *__restrict__ a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (uint32_t)i;
}

// relabel: storage slot p takes user particle vals[p]
__global__ void k_relabel(float4 *__restrict__ dst, const float4 *__restrict__ src_user,
                          const uint32_t *__restrict__ vals, uint32_t *__restrict__ uid, int64_t n) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) {
    uint32_t u = vals[p];
    dst[p] = src_user[u];
    uid[p] = u;
  }
}

// storage-slot state from user-order arrays: pos4[s] = (pos[uid], mass[uid]);
// vel4[s - lo] = vel[uid] for the own range (vel == null -> 0)
__global__ void k_load_state(float4 *__restrict__ pos4, float4 *__restrict__ vel4, const uint32_t *__restrict__ uid,
                             const float *__restrict__ pos, const float *__restrict__ mass,
                             const float *__restrict__ vel, int64_t n, int64_t lo, int64_t hi) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  uint32_t u = uid[s];
  pos4[s] = make_float4(pos[3 * (size_t)u], pos[3 * (size_t)u + 1], pos[3 * (size_t)u + 2],
                        mass ? mass[u] : pos4[s].w);  // no masses: keep the current ones
  if (s >= lo && s < hi)
    vel4[s - lo] = vel ? make_float4(vel[3 * (size_t)u], vel[3 * (size_t)u + 1], vel[3 * (size_t)u + 2], 0.f)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
}

// bh_advance: positions (+ masses, or the current ones) and, later, the own
// slice's velocities, user order -> storage order
__global__ void k_load_pos(float4 *__restrict__ pos4, const uint32_t *__restrict__ uid, const float *__restrict__ pos,
                           const float *__restrict__ mass, int64_t n) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  uint32_t u = uid[s];
  pos4[s] = make_float4(pos[3 * (size_t)u], pos[3 * (size_t)u + 1], pos[3 * (size_t)u + 2], mass ? mass[u] : pos4[s].w);
}
__global__ void k_load_vel(float4 *__restrict__ vel4, const uint32_t *__restrict__ uid, const float *__restrict__ vel,
                           int64_t lo, int64_t hi) {
  int64_t s = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= hi) return;
  uint32_t u = uid[s];
  vel4[s - lo] = vel ? make_float4(vel[3 * (size_t)u], vel[3 * (size_t)u + 1], vel[3 * (size_t)u + 2], 0.f)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
}

// K7 apart (bh_advance's first step): v += a kick, x += v dt, as the walk's
// fused epilogue does it (acc: own slice, storage order, G applied)
struct PeerPtrs {
  int n;
  float4 *p[BH_MAX_PEERS];
};
__global__ void k_kick_drift(float4 *__restrict__ pos4, float4 *__restrict__ vel4, const float *__restrict__ acc,
                             int64_t lo, int64_t hi, float kick, float dt, const PeerPtrs peers) {
  int64_t s = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= hi) return;
  const size_t o = (size_t)(s - lo);
  float4 v = vel4[o];
  v.x = fmaf(acc[3 * o + 0], kick, v.x);
  v.y = fmaf(acc[3 * o + 1], kick, v.y);
  v.z = fmaf(acc[3 * o + 2], kick, v.z);
  vel4[o] = v;
  const float4 x = pos4[s];
  const float4 y = make_float4(fmaf(v.x, dt, x.x), fmaf(v.y, dt, x.y), fmaf(v.z, dt, x.z), x.w);
  pos4[s] = y;
  for (int k = 0; k < peers.n; k++) peers.p[k][s] = y;  // bh_set_peers: the fused exchange
}

// user-order outputs from storage slots [lo, hi): out[uid[s]] = src(s)
// own-slice velocities [k][3] (storage order) -> vel4[k]
__global__ void k_vel3to4(float4 *__restrict__ vel4, const float *__restrict__ v3, int64_t m) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) vel4[k] = make_float4(v3[3 * k], v3[3 * k + 1], v3[3 * k + 2], 0.f);
}
__global__ void k_vel4to3(float *__restrict__ v3, const float4 *__restrict__ vel4, int64_t m) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m) {
    const float4 v = vel4[k];
    v3[3 * k] = v.x;
    v3[3 * k + 1] = v.y;
    v3[3 * k + 2] = v.z;
  }
}

__global__ void k_scatter3(float *__restrict__ out, const float4 *__restrict__ src4, const float *__restrict__ src3,
                           const uint32_t *__restrict__ uid, int64_t lo, int64_t hi, int src_offset_lo) {
  int64_t s = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= hi) return;
  uint32_t u = uid[s];
  int64_t k = src_offset_lo ? s - lo : s;
  if (src4) {
    float4 v = src4[k];
    out[3 * (size_t)u] = v.x; out[3 * (size_t)u + 1] = v.y; out[3 * (size_t)u + 2] = v.z;
  } else {
    out[3 * (size_t)u] = src3[3 * k]; out[3 * (size_t)u + 1] = src3[3 * k + 1]; out[3 * (size_t)u + 2] = src3[3 * k + 2];
  }
}

__global__ void k_scatter1(uint32_t *__restrict__ out, const uint32_t *__restrict__ src, const uint32_t *__restrict__ uid,
                           int64_t lo, int64_t hi) {
  int64_t s = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s < hi) out[uid[s]] = src[s];
}

}  // namespace bh

// ---------------------------------------------------------------- helpers
// eps > 0 as the walk sees it: fp32 eps^2 a normal number (eps >~ 1.1e-19)
static bool eps2_normal(double eps) { return (float)(eps * eps) >= FLT_MIN; }

static unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }

static bh_status validate(const bh_params *p, char *err, size_t errn) {
  if (!p) { snprintf(err, errn, "null params"); return BH_ERR_ARG; }
  if (p->n < 1 || p->n > ((int64_t)1 << 30)) { snprintf(err, errn, "n must be in [1, 2^30]"); return BH_ERR_ARG; }
  if (!(p->theta >= 0.0) || !(p->eps >= 0.0) || !(p->G > 0.0) || !(p->dt > 0.0)) {
    snprintf(err, errn, "need theta >= 0, eps >= 0, G > 0, dt > 0");
    return BH_ERR_ARG;
  }
  if (p->world < 1 || p->rank < 0 || p->rank >= p->world || p->world > p->n) {
    snprintf(err, errn, "need 0 <= rank < world <= n");
    return BH_ERR_ARG;
  }
  if (p->node_capacity != 0 && (p->node_capacity < p->n + 1 || p->node_capacity > BH_MAX_RECORDS)) {
    snprintf(err, errn, "node_capacity must be 0 or in [n + 1, 2^31 - 2]");
    return BH_ERR_ARG;
  }
  if (p->multipole < 0 || p->multipole > 2) {
    snprintf(err, errn, "multipole must be 0, 1 or 2");
    return BH_ERR_ARG;
  }
  int g = p->walk_group;
  if (!(g == 0 || (g >= 66 && g <= 70))) {
    snprintf(err, errn, "walk_group must be 0 (automatic) or 66..70");
    return BH_ERR_ARG;
  }
  return BH_OK;
}

static thread_local char g_err[512];

static cudaEvent_t take_event(bh_ctx *ctx) {
  if (!ctx->free_events.empty()) {
    cudaEvent_t e = ctx->free_events.back();
    ctx->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

static void prof_begin(bh_ctx *ctx, ProfPair *pp, int phase) {
  if (!ctx->prof) return;
  pp->a = take_event(ctx);
  pp->b = take_event(ctx);
  pp->phase = phase;
  pp->launches = 0;
  cudaEventRecord(pp->a, ctx->stream);
}
static void prof_end(bh_ctx *ctx, ProfPair *pp, int launches) {
  if (!ctx->prof) return;
  cudaEventRecord(pp->b, ctx->stream);
  pp->launches = launches;
  ctx->pending.push_back(*pp);
}
static void prof_collect(bh_ctx *ctx) {
  for (auto &pp : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pp.a, pp.b) == cudaSuccess) ctx->prof_ms[pp.phase] += ms;
    ctx->prof_launches[pp.phase] += pp.launches;
    ctx->free_events.push_back(pp.a);
    ctx->free_events.push_back(pp.b);
  }
  ctx->pending.clear();
}

static bh_status status_from_device(bh_ctx *ctx) {
  uint32_t e = ctx->hstatus->err;
  if (e & ERR_NONFINITE_POS) return fail(ctx, BH_ERR_NONFINITE, "non-finite position or mass in the state");
  if (e & ERR_NODE_OVERFLOW)
    return fail(ctx, BH_ERR_OOM, "tree needs %u records (> node_capacity %lld); raise bh_params.node_capacity",
                ctx->hstatus->n_records, (long long)ctx->lay.cap_rec);
  if (e & ERR_NONFINITE_FORCE)
    return fail(ctx, BH_ERR_NONFINITE, "eps == 0 and two particles coincide: infinite force");
  return BH_OK;
}

static bh_status enqueue_status(bh_ctx *ctx) {
  CK(cudaMemcpyAsync(ctx->hstatus, ctx->W.status, sizeof(DevStatus), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaEventRecord(ctx->status_ev, ctx->stream));
  ctx->status_pending = true;
  return BH_OK;
}

static bh_status do_sync(bh_ctx *ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->status_pending) ctx->status_pending = false;
  CK(cudaMemcpy(ctx->hstatus, ctx->W.status, sizeof(DevStatus), cudaMemcpyDeviceToHost));
  if (ctx->prof) prof_collect(ctx);
  return status_from_device(ctx);
}

static bh_status set_dev(bh_ctx *ctx) {
  CK(cudaSetDevice(ctx->p.device));
  return BH_OK;
}

// K0-K5 on the current pos4
static bh_status build_tree(bh_ctx *ctx) {
  const int64_t n = ctx->p.n;
  cudaStream_t s = ctx->stream;
  ProfPair pp;
  // clear per-build counters (interactions/fallbacks are per walk)
  prof_begin(ctx, &pp, 0);
  CK(launch_bbox(ctx->W, n, s));
  prof_end(ctx, &pp, 1);
  // K1 + K2: the near-sorted path from the previous build's order, else (its
  // device flag cleared) K1 and the full radix sort
  prof_begin(ctx, &pp, 1);
  int buf = 0;
  if (ctx->near_sort) CK(launch_near_sort(ctx->W, n, s));
  CK(launch_keys(ctx->W, n, s));
  CK(launch_sort(ctx->W, n, s, &buf));
  // (equal keys are ordered by user index in K4's first kernel, k_lcp_count)
  prof_end(ctx, &pp, (ctx->near_sort ? 22 : 0) + 2 + SORT_PASSES + 1);  // (+ zeroing, - tie fix-up)
  ctx->sort_buf = buf;
  prof_begin(ctx, &pp, 2);
  CK(launch_tree(ctx->W, n, ctx->lay.cap_rec, buf, ctx->cont_fold, s));  // (zeroes the particles' quadrupoles)
  prof_end(ctx, &pp, 8);
  prof_begin(ctx, &pp, 3);
  int launches = 0;
  CK(launch_moments(ctx->W, n, ctx->p.theta, (float)(ctx->p.eps * ctx->p.eps), ctx->cont_fold, s, &launches));
  prof_end(ctx, &pp, launches);
  ctx->tree_valid = true;
  return BH_OK;
}

static bh_status walk(bh_ctx *ctx, int mode, float kick, float *acc_out, bool user_order) {
  const int64_t n = ctx->p.n;
  cudaStream_t s = ctx->stream;
  ProfPair pp;
  prof_begin(ctx, &pp, 4);
  int launches = 1;
  WalkArgs a;
  memset(&a, 0, sizeof a);
  a.n = n;
  a.buf = ctx->sort_buf;
  // walk_group 0 = automatic (measured on the BASELINE configs):
  // 4 targets per lane from 2^19 particles (half the record bytes per
  // target-visit) -- 8-target groups of 2 lanes (code 69) for long walks
  // (theta < 0.6: ~2000 interactions per target, cfg4) and up to 2^22 (cfg3),
  // one lane's own 4 targets (code 70) for shorter walks on n >= 2^22 (cfg5);
  // below 2^19 (launch-bound sizes) 2 lanes x 2 targets (code 68)
  // (multipole = 2 keeps 2 targets per lane: its quadrupole terms fill the
  // registers -- 4 per lane measured 117 vs 95 ms on cfg4)
  const int64_t nn = n;
  const bool quad = ctx->p.multipole == 2;
  const int auto_group = quad ? ((ctx->p.theta < 0.6 && nn >= ((int64_t)1 << 22)) ? 67 : 68)
                         : nn >= ((int64_t)1 << 22) ? (ctx->p.theta < 0.6 ? 69 : 70)
                         : nn >= ((int64_t)1 << 19) ? 69 : 68;
  a.group = ctx->p.walk_group != 0 ? ctx->p.walk_group : auto_group;
  a.stats = ctx->walk_stats;
  a.num_sms = ctx->num_sms;
  // containment test elision (see walk.cu): a cell holding the target has
  // s/d >= 1/sqrt(3) (d <= sqrt(3) s), so it never passes s/d < theta for
  // theta < 0.5773; kept with a margin, and only when eps > 0 -- as the walk's
  // fp32 eps^2, a normal float, so every unmasked force is finite (rsqrt of a
  // zero or flushed-denormal r2 would be inf, and 0 x inf a NaN)
  a.need_cont = !(ctx->p.theta < 0.57 && eps2_normal(ctx->p.eps)) && !ctx->cont_fold;
  a.mode = mode;
  a.eps2 = (float)(ctx->p.eps * ctx->p.eps);
  a.G = (float)ctx->p.G;
  a.kick = kick;
  a.dt = (float)ctx->p.dt;
  a.theta2 = ctx->p.theta * ctx->p.theta;
  a.quad = ctx->p.multipole == 2;
  a.own_lo = (uint32_t)ctx->own_lo;
  a.own_hi = (uint32_t)ctx->own_hi;
  a.acc_out = mode == 0 ? acc_out : nullptr;
  a.user_order = user_order ? 1 : 0;
  a.n_peers = (int)ctx->peers.size();
  a.peer_pos4 = ctx->peers.data();
  CK(cudaMemsetAsync(&ctx->W.status->interactions, 0, 6 * sizeof(unsigned long long), s));
  // world > 1: the rank walks the P = 1 groups that hold one of its particles
  // (every target summed in the same group as at P = 1: bitwise equal results)
  a.own_check = ctx->p.world > 1 ? 1 : 0;
  if (a.own_check) launches += 4;
  CK(launch_walk(ctx->W, a, s));
  prof_end(ctx, &pp, launches);
  ctx->walked = true;
  return BH_OK;
}

// bh_set_peers with a communicator: a one-word all-reduce orders the ranks'
// phases (every replica written before anyone builds from it; nobody writes a
// replica its owner still reads)
static bh_status peer_barrier(bh_ctx *ctx) {
  if (ctx->peers.empty() || !ctx->p.nccl_comm) return BH_OK;
  uint32_t *w = &ctx->W.status->pad[0];
  ncclResult_t rc = ncclAllReduce(w, w, 1, ncclUint32, ncclMax, (ncclComm_t)ctx->p.nccl_comm, ctx->stream);
  if (rc != ncclSuccess) return fail(ctx, BH_ERR_NCCL, "ncclAllReduce (barrier): %s", ncclGetErrorString(rc));
  return BH_OK;
}

static bh_status exchange(bh_ctx *ctx) {
  if (ctx->p.world == 1) return BH_OK;
  if (!ctx->peers.empty()) {  // K8 rode on K7's stores: only the barrier is left
    ProfPair pp;
    prof_begin(ctx, &pp, 5);
    bh_status st = peer_barrier(ctx);
    if (st) return st;
    prof_end(ctx, &pp, ctx->p.nccl_comm ? 1 : 0);
    return BH_OK;
  }
  if (!ctx->p.nccl_comm) return BH_OK;
  ProfPair pp;
  prof_begin(ctx, &pp, 5);
  ncclComm_t comm = (ncclComm_t)ctx->p.nccl_comm;
  const int64_t n = ctx->p.n;
  const int P = ctx->p.world;
  if (ncclGroupStart() != ncclSuccess) return fail(ctx, BH_ERR_NCCL, "ncclGroupStart failed");
  (void)n;
  for (int r = 0; r < P; r++) {
    const int64_t lo = ctx->bounds[r], hi = ctx->bounds[r + 1];
    if (hi <= lo) continue;
    float *buf = (float *)(ctx->W.pos4 + lo);
    ncclResult_t rc = ncclBroadcast(buf, buf, (size_t)(hi - lo) * 4, ncclFloat, r, comm, ctx->stream);
    if (rc != ncclSuccess) {
      ncclGroupEnd();
      return fail(ctx, BH_ERR_NCCL, "ncclBroadcast: %s", ncclGetErrorString(rc));
    }
  }
  ncclResult_t rc = ncclGroupEnd();
  if (rc != ncclSuccess) return fail(ctx, BH_ERR_NCCL, "ncclGroupEnd: %s", ncclGetErrorString(rc));
  prof_end(ctx, &pp, 1);
  return BH_OK;
}

// copy caller inputs (user order) into device scratch: pos -> accu, mass -> targets,
// vel -> the record region; returns device pointers
static bh_status stage_inputs(bh_ctx *ctx, const float *mass, const float *pos, const float *vel, int where,
                              const float **dm, const float **dp, const float **dv) {
  const int64_t n = ctx->p.n;
  if (where == BH_DEVICE) {
    *dm = mass; *dp = pos; *dv = vel;
    return BH_OK;
  }
  float *sp = ctx->W.accu;
  float *sm = (float *)ctx->W.targets;
  float *sv = (float *)ctx->W.rec;
  CK(cudaMemcpyAsync(sp, pos, (size_t)n * 12, cudaMemcpyHostToDevice, ctx->stream));
  if (mass) CK(cudaMemcpyAsync(sm, mass, (size_t)n * 4, cudaMemcpyHostToDevice, ctx->stream));
  if (vel) CK(cudaMemcpyAsync(sv, vel, (size_t)n * 12, cudaMemcpyHostToDevice, ctx->stream));
  *dm = mass ? sm : nullptr; *dp = sp; *dv = vel ? sv : nullptr;
  return BH_OK;
}

// ---------------------------------------------------------------- ABI
extern "C" {

size_t bh_workspace_bytes(const bh_params *p) {
  char e[128];
  if (validate(p, e, sizeof e) != BH_OK) return 0;
  return make_layout(p->n, p->world, p->node_capacity, p->multipole).total;
}

const char *bh_status_string(int st) {
  switch (st) {
    case BH_OK: return "BH_OK";
    case BH_ERR_ARG: return "BH_ERR_ARG";
    case BH_ERR_CUDA: return "BH_ERR_CUDA";
    case BH_ERR_OOM: return "BH_ERR_OOM";
    case BH_ERR_STATE: return "BH_ERR_STATE";
    case BH_ERR_NONFINITE: return "BH_ERR_NONFINITE";
    case BH_ERR_NCCL: return "BH_ERR_NCCL";
    default: return "BH_UNKNOWN";
  }
}

const char *bh_last_error(const bh_ctx *ctx) { return ctx ? ctx->err : g_err; }

bh_status bh_create(bh_ctx **out, const bh_params *p, const float *mass, const float *pos, const float *vel,
                    int where) {
  if (!out) { snprintf(g_err, sizeof g_err, "null out"); return BH_ERR_ARG; }
  *out = nullptr;
  bh_status v = validate(p, g_err, sizeof g_err);
  if (v != BH_OK) return v;
  if (!mass || !pos || (where != BH_HOST && where != BH_DEVICE)) {
    snprintf(g_err, sizeof g_err, "need mass, pos and where in {BH_HOST, BH_DEVICE}");
    return BH_ERR_ARG;
  }
  Layout lay = make_layout(p->n, p->world, p->node_capacity, p->multipole);
  if (!p->workspace || p->workspace_bytes < lay.total || ((uintptr_t)p->workspace & 255)) {
    snprintf(g_err, sizeof g_err, "workspace must be 256-aligned and >= %zu bytes", lay.total);
    return BH_ERR_OOM;
  }
  bh_ctx *ctx = new bh_ctx();
  ctx->p = *p;
  ctx->lay = lay;
  ctx->err[0] = 0;
  ctx->prof = false;
  ctx->prof_calls = 0;
  memset(ctx->prof_ms, 0, sizeof ctx->prof_ms);
  memset(ctx->prof_launches, 0, sizeof ctx->prof_launches);
  bind_workspace(lay, p->workspace, ctx->W);
  // test hooks: a smaller resume-state capacity / resume stack exercises the
  // walk's rare paths (queue slots restarting from the root, stack overflow)
  if (getenv("BH_RESUME_CAP")) {
    const long long c = atoll(getenv("BH_RESUME_CAP"));
    if (c >= 0 && c < ctx->W.cap_resume) ctx->W.cap_resume = c;
  }
  ctx->W.resume_stack = getenv("BH_RESUME_STACK") ? atoi(getenv("BH_RESUME_STACK")) : 0;
  const int64_t n = p->n;
  ctx->own_lo = n * p->rank / p->world;
  ctx->own_hi = n * (p->rank + 1) / p->world;
  ctx->bounds.resize((size_t)p->world + 1);
  for (int r = 0; r <= p->world; r++) ctx->bounds[r] = n * r / p->world;
  ctx->steps = 0;
  ctx->tree_valid = false;
  ctx->walked = false;
  ctx->walk_stats = 0;
  ctx->use_graphs = getenv("BH_NO_GRAPHS") ? 0 : 1;
  // the near-sorted path pays for its ~20 launches from ~2^18 particles on
  // (measured: cfg2, 2^16, 2% slower with it; cfg3, 2^20, 7% faster)
  ctx->cont_fold = (p->theta >= 0.57 && eps2_normal(p->eps) && !getenv("BH_NO_CONT_FOLD")) ? 1 : 0;
  ctx->near_sort = getenv("BH_NO_NEAR_SORT") ? 0 : (p->n >= ((int64_t)1 << 18) || getenv("BH_NEAR_SORT") ? 1 : 0);
  ctx->step_graph[0] = ctx->step_graph[1] = ctx->step_graph[2] = nullptr;
  ctx->num_sms = 148;
  ctx->sort_buf = 0;
  ctx->status_pending = false;
  ctx->io_stream = nullptr;
  ctx->io_ev_pos = ctx->io_ev_vel = nullptr;
  ctx->vel_pending = false;
  ctx->vel_src = nullptr;
  bh_status st = BH_OK;
  do {
    if (cudaSetDevice(p->device) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "cudaSetDevice(%d) failed", p->device); break; }
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, p->device);
    if (ctx->num_sms < 1 || ctx->num_sms > 256) ctx->num_sms = 148;
    if (p->stream) {
      ctx->stream = (cudaStream_t)p->stream;
      ctx->own_stream = false;
    } else {
      if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "stream create failed"); break; }
      ctx->own_stream = true;
    }
    if (cudaMallocHost(&ctx->hstatus, sizeof(DevStatus)) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "pinned alloc failed"); break; }
    if (cudaEventCreateWithFlags(&ctx->status_ev, cudaEventDisableTiming) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "event create failed"); break; }
    cudaStream_t s = ctx->stream;
    if (cudaMemsetAsync(ctx->W.status, 0, sizeof(DevStatus), s) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "memset failed"); break; }
    const float *dm, *dp, *dv;
    st = stage_inputs(ctx, mass, pos, vel, where, &dm, &dp, &dv);
    if (st) break;
    // user-order pos4 -> step-0 Morton order -> storage order
    k_pack<<<blocks_for(n), 256, 0, s>>>(ctx->W.pos4, dp, dm, n);
    k_iota<<<blocks_for(n), 256, 0, s>>>(ctx->W.uid, n);
    if (cudaGetLastError() != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "pack launch failed"); break; }
    // velocities (user order) parked as float4 in lvl_mom (>= 32 B per particle)
    float4 *vtmp = (float4 *)ctx->W.lvl_mom;
    if (dv) {
      k_pack<<<blocks_for(n), 256, 0, s>>>(vtmp, dv, dm, n);  // .w = mass, ignored
    }
    if (launch_bbox(ctx->W, n, s) != cudaSuccess || launch_keys(ctx->W, n, s) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "keys launch failed"); break; }
    int buf = 0;
    if (launch_sort(ctx->W, n, s, &buf) != cudaSuccess || launch_tie_fixup(ctx->W, n, buf, s) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "sort launch failed"); break; }
    // relabel: gather user-order pos4 into the record scratch, copy back; uid[p] = user index
    float4 *scratch = (float4 *)ctx->W.rec;
    k_relabel<<<blocks_for(n), 256, 0, s>>>(scratch, ctx->W.pos4, ctx->W.vals[buf], ctx->W.uid, n);
    if (cudaMemcpyAsync(ctx->W.pos4, scratch, (size_t)n * 16, cudaMemcpyDeviceToDevice, s) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "copy failed"); break; }
    int64_t own_n = ctx->own_hi - ctx->own_lo;
    if (dv) {
      // vel4[s - lo] = vtmp[uid[s]] for own s: relabel into the scratch then copy the own slice
      k_relabel<<<blocks_for(n), 256, 0, s>>>(scratch, vtmp, ctx->W.vals[buf], ctx->W.uid, n);
      if (cudaMemcpyAsync(ctx->W.vel4, scratch + ctx->own_lo, (size_t)own_n * 16, cudaMemcpyDeviceToDevice, s) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "copy failed"); break; }
    } else {
      if (cudaMemsetAsync(ctx->W.vel4, 0, (size_t)own_n * 16, s) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "memset failed"); break; }
    }
    if (cudaMemsetAsync(ctx->W.icount, 0, (size_t)n * 4, s) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "memset failed"); break; }
    // storage order is the step-0 Morton order: the previous order of the first
    // build's near-sorted path is the identity (vals[0] always holds a permutation)
    k_iota<<<blocks_for(n), 256, 0, s>>>(ctx->W.vals[0], n);
    if (cudaMemsetAsync(ctx->W.gcost, 0, (size_t)n * 4, s) != cudaSuccess) { st = fail(ctx, BH_ERR_CUDA, "memset failed"); break; }
    st = do_sync(ctx);
  } while (0);
  if (st != BH_OK) {
    snprintf(g_err, sizeof g_err, "%s", ctx->err);
    bh_destroy(ctx);
    return st;
  }
  *out = ctx;
  return BH_OK;
}

bh_status bh_set_state(bh_ctx *ctx, const float *mass, const float *pos, const float *vel, int where) {
  if (!ctx || !pos || (where != BH_HOST && where != BH_DEVICE)) return fail(ctx, BH_ERR_ARG, "bad arguments");
  bh_status st = set_dev(ctx);
  if (st) return st;
  const int64_t n = ctx->p.n;
  const float *dm, *dp, *dv;
  st = stage_inputs(ctx, mass, pos, vel, where, &dm, &dp, &dv);
  if (st) return st;
  k_load_state<<<blocks_for(n), 256, 0, ctx->stream>>>(ctx->W.pos4, ctx->W.vel4, ctx->W.uid, dp, dm, dv, n,
                                                        ctx->own_lo, ctx->own_hi);
  ctx->vel_pending = false;  // (a pending bh_advance upload is superseded)
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(&ctx->W.status->err, 0, sizeof(uint32_t), ctx->stream));
  ctx->steps = 0;
  ctx->tree_valid = false;
  return BH_OK;
}

bh_status bh_build_tree(bh_ctx *ctx) {
  if (!ctx) return BH_ERR_ARG;
  bh_status st = set_dev(ctx);
  if (st) return st;
  if (ctx->prof) ctx->prof_calls++;
  st = build_tree(ctx);
  if (st) return st;
  return enqueue_status(ctx);
}

bh_status bh_compute_forces(bh_ctx *ctx, float *acc, int where) {
  if (!ctx || (where != BH_HOST && where != BH_DEVICE)) return fail(ctx, BH_ERR_ARG, "bad arguments");
  if (!ctx->tree_valid) return fail(ctx, BH_ERR_STATE, "bh_compute_forces needs bh_build_tree on the current state");
  bh_status st = set_dev(ctx);
  if (st) return st;
  const int64_t lo = ctx->own_lo, hi = ctx->own_hi, own_n = hi - lo;
  const bool host_scatter = acc && where == BH_HOST && ctx->p.world > 1;
  // device destination: the walk writes user order directly; host + one rank:
  // user order into accu then one copy; host + several ranks: storage order + host scatter
  float *dst = !acc ? nullptr : (where == BH_DEVICE ? acc : ctx->W.accu);
  st = walk(ctx, 0, 0.f, dst, !host_scatter);
  if (st) return st;
  if (!acc) return enqueue_status(ctx);
  if (where == BH_DEVICE) return enqueue_status(ctx);
  if (!host_scatter) {
    CK(cudaMemcpyAsync(acc, ctx->W.accu, (size_t)ctx->p.n * 12, cudaMemcpyDeviceToHost, ctx->stream));
    return do_sync(ctx);
  }
  std::vector<float> a((size_t)own_n * 3);
  std::vector<uint32_t> u((size_t)own_n);
  CK(cudaMemcpyAsync(a.data(), ctx->W.accu, (size_t)own_n * 12, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(u.data(), ctx->W.uid + lo, (size_t)own_n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  st = do_sync(ctx);
  if (st) return st;
  for (int64_t k = 0; k < own_n; k++) {
    size_t ui = u[k];
    acc[3 * ui] = a[3 * k]; acc[3 * ui + 1] = a[3 * k + 1]; acc[3 * ui + 2] = a[3 * k + 2];
  }
  return BH_OK;
}

// one time step's launches (K0-K8) on ctx->stream
// bh_advance's velocities: wait for their upload and load the own slice
static bh_status flush_vel(bh_ctx *ctx) {
  if (!ctx->vel_pending) return BH_OK;
  // (inside graph [2] the event was recorded outside the capture: an external wait node)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(ctx->stream, &cs));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->io_ev_vel, cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0));
  const int64_t own_n = ctx->own_hi - ctx->own_lo;
  k_load_vel<<<blocks_for(own_n), 256, 0, ctx->stream>>>(ctx->W.vel4, ctx->W.uid, ctx->vel_src, ctx->own_lo,
                                                          ctx->own_hi);
  CK(cudaGetLastError());
  ctx->vel_pending = false;
  return BH_OK;
}

static bh_status enqueue_walk(bh_ctx *ctx, float kick);
static bh_status enqueue_step(bh_ctx *ctx, float kick) {
  bh_status st = build_tree(ctx);
  if (st) return st;
  // bh_set_peers: every rank has finished reading its replica before any K7
  // writes into it
  st = peer_barrier(ctx);
  if (st) return st;
  return enqueue_walk(ctx, kick);
}

// K6-K8 of a step on the tree just built
static bh_status enqueue_walk(bh_ctx *ctx, float kick) {
  bh_status st = BH_OK;
  if (ctx->vel_pending) {
    // first step of bh_advance: the walk computes forces (own slice, storage
    // order) while the velocity upload finishes, then K7 runs apart with the
    // walk epilogue's exact operations (finish() in walk_common.cuh)
    st = walk(ctx, 0, 0.f, ctx->W.accu, false);
    if (st) return st;
    st = flush_vel(ctx);
    if (st) return st;
    const int64_t own_n = ctx->own_hi - ctx->own_lo;
    PeerPtrs pp;
    pp.n = (int)ctx->peers.size();
    for (int k = 0; k < BH_MAX_PEERS; k++) pp.p[k] = k < pp.n ? ctx->peers[k] : nullptr;
    k_kick_drift<<<blocks_for(own_n), 256, 0, ctx->stream>>>(ctx->W.pos4, ctx->W.vel4, ctx->W.accu, ctx->own_lo,
                                                              ctx->own_hi, kick, (float)ctx->p.dt, pp);
    CK(cudaGetLastError());
  } else {
    st = walk(ctx, 1, kick, nullptr, false);
  }
  if (st) return st;
  return exchange(ctx);
}

static void drop_graphs(bh_ctx *ctx) {
  for (int i = 0; i < 3; i++)
    if (ctx->step_graph[i]) {
      cudaGraphExecDestroy(ctx->step_graph[i]);
      ctx->step_graph[i] = nullptr;
    }
}

// The step is a fixed sequence of ~45 launches whose sizes do not depend on the
// data (every kernel reads its counts from the device), so it is captured once
// per kick value into a CUDA graph and replayed: one launch per step instead of
// ~45 (matters for the small configurations).  Not used while profiling (the
// per-phase events).  With an NCCL communicator the grouped broadcast of K8 is
// captured too (NCCL supports stream capture); bh_set_partition drops the
// graphs, since the ranges are baked in.
static bh_status step_graph(bh_ctx *ctx, int which, float kick, cudaGraphExec_t *out) {
  if (ctx->step_graph[which]) {
    *out = ctx->step_graph[which];
    return BH_OK;
  }
  cudaGraph_t g = nullptr;
  // [2] captures the velocity load of bh_advance (a wait on io_ev_vel, recorded
  // outside the graph, then k_load_vel from vstage) between build and walk
  const bool pending = ctx->vel_pending;
  ctx->vel_pending = which == 2;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  bh_status st = enqueue_step(ctx, kick);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  ctx->vel_pending = pending;
  if (st) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (e != cudaSuccess) return fail(ctx, BH_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&ctx->step_graph[which], g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    ctx->step_graph[which] = nullptr;
    return fail(ctx, BH_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
  }
  *out = ctx->step_graph[which];
  return BH_OK;
}

// bh_set_peers without a communicator: nothing inside a step orders this rank's
// K7 stores after the other ranks' builds, so only bh_step_phase may step
static bool peers_unordered(const bh_ctx *ctx) { return !ctx->peers.empty() && !ctx->p.nccl_comm; }

bh_status bh_step(bh_ctx *ctx, int nsteps) {
  if (!ctx || nsteps < 0) return fail(ctx, BH_ERR_ARG, "bad arguments");
  if (nsteps > 0 && peers_unordered(ctx))
    return fail(ctx, BH_ERR_STATE, "bh_set_peers without an NCCL communicator: step with bh_step_phase");
  bh_status st = set_dev(ctx);
  if (st) return st;
  if (ctx->status_pending && cudaEventQuery(ctx->status_ev) == cudaSuccess) {
    ctx->status_pending = false;
    st = status_from_device(ctx);
    if (st) return st;
  }
  for (int k = 0; k < nsteps; k++) {
    // (a captured step must not contain bh_advance's one-off velocity load)
    // (with NCCL the captured step holds the grouped broadcast too; a capture
    // the NCCL build refuses switches graphs off for this ctx: direct launches)
    const bool graphs = ctx->use_graphs && !ctx->prof && !ctx->vel_pending;
    if (ctx->prof) ctx->prof_calls++;
    const int which = ctx->steps == 0 ? 0 : 1;
    const float kick = (float)(which == 0 ? 0.5 * ctx->p.dt : ctx->p.dt);
    cudaGraphExec_t ge = nullptr;
    if (graphs) {
      st = step_graph(ctx, which, kick, &ge);
      if (st && ctx->p.world > 1 && ctx->p.nccl_comm) {  // NCCL refused capture
        cudaGetLastError();
        ctx->use_graphs = 0;
        ge = nullptr;
        st = BH_OK;
      }
      if (st) return st;
    }
    if (ge) {
      CK(cudaGraphLaunch(ge, ctx->stream));
      ctx->sort_buf = 0;  // 8 passes: the sorted keys end in buffer 0
    } else {
      st = enqueue_step(ctx, kick);
      if (st) return st;
    }
    ctx->steps++;
    ctx->tree_valid = false;
  }
  return enqueue_status(ctx);
}

bh_status bh_sync(bh_ctx *ctx) {
  if (!ctx) return BH_ERR_ARG;
  bh_status st = set_dev(ctx);
  if (st) return st;
  return do_sync(ctx);
}

bh_status bh_destroy(bh_ctx *ctx) {
  if (!ctx) return BH_OK;
  cudaSetDevice(ctx->p.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (auto &pp : ctx->pending) { cudaEventDestroy(pp.a); cudaEventDestroy(pp.b); }
  for (auto e : ctx->free_events) cudaEventDestroy(e);
  drop_graphs(ctx);
  if (ctx->status_ev) cudaEventDestroy(ctx->status_ev);
  if (ctx->io_stream) cudaStreamSynchronize(ctx->io_stream);
  if (ctx->io_ev_pos) cudaEventDestroy(ctx->io_ev_pos);
  if (ctx->io_ev_vel) cudaEventDestroy(ctx->io_ev_vel);
  if (ctx->io_stream) cudaStreamDestroy(ctx->io_stream);
  if (ctx->hstatus) cudaFreeHost(ctx->hstatus);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return BH_OK;
}

bh_status bh_get_state(bh_ctx *ctx, float *pos, float *vel, int where) {
  if (!ctx || (where != BH_HOST && where != BH_DEVICE)) return fail(ctx, BH_ERR_ARG, "bad arguments");
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = flush_vel(ctx);
  if (st) return st;
  const int64_t n = ctx->p.n, lo = ctx->own_lo, hi = ctx->own_hi, own_n = hi - lo;
  cudaStream_t s = ctx->stream;
  if (pos) {
    float *dst = where == BH_DEVICE ? pos : ctx->W.accu;
    k_scatter3<<<blocks_for(n), 256, 0, s>>>(dst, ctx->W.pos4, nullptr, ctx->W.uid, 0, n, 0);
    CK(cudaGetLastError());
    if (where == BH_HOST) CK(cudaMemcpyAsync(pos, ctx->W.accu, (size_t)n * 12, cudaMemcpyDeviceToHost, s));
  }
  if (vel) {
    if (where == BH_DEVICE) {
      k_scatter3<<<blocks_for(own_n), 256, 0, s>>>(vel, ctx->W.vel4, nullptr, ctx->W.uid, lo, hi, 1);
      CK(cudaGetLastError());
    } else if (ctx->p.world == 1) {
      float *tmp = ctx->W.accu;  // stream order: the position copy above has finished reading it
      k_scatter3<<<blocks_for(own_n), 256, 0, s>>>(tmp, ctx->W.vel4, nullptr, ctx->W.uid, lo, hi, 1);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(vel, tmp, (size_t)n * 12, cudaMemcpyDeviceToHost, s));
    } else {
      std::vector<float4> v((size_t)own_n);
      std::vector<uint32_t> u((size_t)own_n);
      CK(cudaMemcpyAsync(v.data(), ctx->W.vel4, (size_t)own_n * 16, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(u.data(), ctx->W.uid + lo, (size_t)own_n * 4, cudaMemcpyDeviceToHost, s));
      st = do_sync(ctx);
      if (st) return st;
      for (int64_t k = 0; k < own_n; k++) {
        size_t ui = u[k];
        vel[3 * ui] = v[k].x; vel[3 * ui + 1] = v[k].y; vel[3 * ui + 2] = v[k].z;
      }
    }
  }
  return do_sync(ctx);
}

// set_state + step(nsteps) + get_state in one call: the velocities (needed
// only by the first walk's leapfrog) are uploaded on a second stream while the
// first tree is built, after the positions' upload (both share the link).
bh_status bh_advance(bh_ctx *ctx, const float *mass, const float *pos, const float *vel, int nsteps, float *pos_out,
                     float *vel_out, int where) {
  if (!ctx || !pos || nsteps < 0 || (where != BH_HOST && where != BH_DEVICE))
    return fail(ctx, BH_ERR_ARG, "bad arguments");
  if (nsteps > 0 && peers_unordered(ctx))
    return fail(ctx, BH_ERR_STATE, "bh_set_peers without an NCCL communicator: step with bh_step_phase");
  bh_status st = set_dev(ctx);
  if (st) return st;
  if (!ctx->io_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->io_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->io_ev_pos, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->io_ev_vel, cudaEventDisableTiming));
  }
  const int64_t n = ctx->p.n;
  cudaStream_t s = ctx->stream;
  const float *dp = pos, *dm = mass;
  if (where == BH_HOST) {
    CK(cudaMemcpyAsync(ctx->W.accu, pos, (size_t)n * 12, cudaMemcpyHostToDevice, s));
    if (mass) CK(cudaMemcpyAsync(ctx->W.targets, mass, (size_t)n * 4, cudaMemcpyHostToDevice, s));
    dp = ctx->W.accu;
    dm = mass ? (const float *)ctx->W.targets : nullptr;
  }
  // the velocity upload starts once the positions are in (and after every
  // earlier use of its staging buffer: the event follows all prior work); it
  // always lands in vstage (device inputs are copied, none = zeros), so the
  // captured first step reads a fixed buffer
  CK(cudaEventRecord(ctx->io_ev_pos, s));
  CK(cudaStreamWaitEvent(ctx->io_stream, ctx->io_ev_pos, 0));
  if (vel) {
    CK(cudaMemcpyAsync(ctx->W.vstage, vel, (size_t)n * 12,
                       where == BH_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->io_stream));
  } else {
    CK(cudaMemsetAsync(ctx->W.vstage, 0, (size_t)n * 12, ctx->io_stream));
  }
  CK(cudaEventRecord(ctx->io_ev_vel, ctx->io_stream));
  ctx->vel_src = ctx->W.vstage;
  ctx->vel_pending = true;
  k_load_pos<<<blocks_for(n), 256, 0, s>>>(ctx->W.pos4, ctx->W.uid, dp, dm, n);
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(&ctx->W.status->err, 0, sizeof(uint32_t), s));
  ctx->steps = 0;
  ctx->tree_valid = false;
  if (nsteps == 0) {
    st = flush_vel(ctx);
  } else {
    // the first step (its velocity load sits between build and walk) as its
    // own captured graph, the rest via bh_step
    if (ctx->prof) ctx->prof_calls++;
    const float kick = (float)(0.5 * ctx->p.dt);
    cudaGraphExec_t ge = nullptr;
    if (ctx->use_graphs && !ctx->prof) {
      st = step_graph(ctx, 2, kick, &ge);
      if (st && ctx->p.world > 1 && ctx->p.nccl_comm) {  // NCCL refused capture
        cudaGetLastError();
        ctx->use_graphs = 0;
        ge = nullptr;
        st = BH_OK;
      }
      if (st) return st;
    }
    if (ge) {
      CK(cudaGraphLaunch(ge, s));
      ctx->sort_buf = 0;
      ctx->vel_pending = false;
    } else {
      st = enqueue_step(ctx, kick);
      if (st) return st;
    }
    ctx->steps++;
    ctx->tree_valid = false;
    st = bh_step(ctx, nsteps - 1);
  }
  if (st) return st;
  // the caller's input buffers are borrowed only for this call
  if (ctx->io_stream) CK(cudaStreamSynchronize(ctx->io_stream));
  if (pos_out || vel_out) return bh_get_state(ctx, pos_out, vel_out, where);
  return do_sync(ctx);
}

bh_status bh_get_root(bh_ctx *ctx, float *lo3, float *L, float *scale) {
  if (!ctx) return BH_ERR_ARG;
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = do_sync(ctx);
  if (st) return st;
  for (int a = 0; a < 3; a++) if (lo3) lo3[a] = ctx->hstatus->lo[a];
  if (L) *L = ctx->hstatus->L;
  if (scale) *scale = ctx->hstatus->scale;
  return BH_OK;
}

bh_status bh_get_keys(bh_ctx *ctx, uint64_t *keys, uint32_t *perm) {
  if (!ctx) return BH_ERR_ARG;
  bh_status st = set_dev(ctx);
  if (st) return st;
  const int64_t n = ctx->p.n;
  cudaStream_t s = ctx->stream;
  if (keys) CK(cudaMemcpyAsync(keys, ctx->W.keys[ctx->sort_buf], (size_t)n * 8, cudaMemcpyDeviceToHost, s));
  if (perm) {
    std::vector<uint32_t> v((size_t)n), u((size_t)n);
    CK(cudaMemcpyAsync(v.data(), ctx->W.vals[ctx->sort_buf], (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(u.data(), ctx->W.uid, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    st = do_sync(ctx);
    if (st) return st;
    for (int64_t p = 0; p < n; p++) perm[p] = u[v[p]];
    return BH_OK;
  }
  return do_sync(ctx);
}

// Level (0 .. 22; 22 = bucket member) and leaf flag of every record, from the
// level-ordered items of K4 (record -> item -> the level whose item range holds
// it; leaf = the item is a particle's own record).  Host side, inspection only.
static bh_status record_levels(bh_ctx *ctx, uint32_t nrec, std::vector<uint8_t> &lev, std::vector<uint8_t> &leaf) {
  std::vector<uint32_t> item(nrec), irec(nrec);
  CK(cudaMemcpy(item.data(), ctx->W.rec_item, (size_t)nrec * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(irec.data(), ctx->W.item_rec, (size_t)nrec * 4, cudaMemcpyDeviceToHost));
  lev.assign(nrec, 0);
  leaf.assign(nrec, 0);
  const uint32_t *off = ctx->hstatus->lvl_offset;
  for (uint32_t c = 0; c < nrec; c++) {
    const uint32_t it = item[c];
    int l = 0;
    while (l + 1 < BH_NLEVELS && off[l + 1] <= it) l++;
    lev[c] = (uint8_t)l;
    leaf[c] = (irec[it] & ITEM_LEAF) ? 1 : 0;
  }
  return BH_OK;
}

static bh_status export_tree(bh_ctx *ctx, uint8_t *level, uint32_t *first, uint32_t *count, double *M, double *MX,
                             int64_t cap, int64_t *n_nodes) {
  // copy the raw records back and re-format on the host (inspection only):
  // drop bucket-member records, count = first(skip) - first, leaf moments (m, m x)
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = do_sync(ctx);
  if (st) return st;
  const int64_t n = ctx->p.n;
  const uint32_t nrec = ctx->hstatus->n_records;
  std::vector<Rec> rec(nrec);
  std::vector<uint32_t> fst(nrec);
  std::vector<double4> mom;
  CK(cudaMemcpy(rec.data(), ctx->W.rec, (size_t)nrec * sizeof(Rec), cudaMemcpyDeviceToHost));
  {  // first particle of each record: particle p owns records [nstart[p], nstart[p+1])
    std::vector<uint32_t> ns((size_t)n + 1);
    CK(cudaMemcpy(ns.data(), ctx->W.nstart, ((size_t)n + 1) * 4, cudaMemcpyDeviceToHost));
    for (int64_t p = 0; p < n; p++)
      for (uint32_t c = ns[p]; c < ns[p + 1] && c < nrec; c++) fst[c] = (uint32_t)p;
  }
  if (M || MX) {
    mom.resize(nrec);
    // fp64 moments: the level-ordered item of each record
    std::vector<uint32_t> item(nrec);
    std::vector<double4> lm(nrec);
    CK(cudaMemcpy(item.data(), ctx->W.rec_item, (size_t)nrec * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(lm.data(), ctx->W.lvl_mom, (size_t)nrec * 32, cudaMemcpyDeviceToHost));
    for (uint32_t c = 0; c < nrec; c++) mom[c] = lm[item[c]];
  }
  std::vector<uint8_t> lev, leafv;
  st = record_levels(ctx, nrec, lev, leafv);
  if (st) return st;
  int64_t k = 0;
  for (uint32_t c = 0; c < nrec; c++) {
    const uint4 a = rec[c].aux;
    if (lev[c] > BH_MAXLEVEL) continue;  // a bucket member (level 22) is not a node of the export
    if (k < cap) {
      const bool leaf = leafv[c] != 0;
      if (level) level[k] = lev[c];
      if (first) first[k] = fst[c];
      if (count) count[k] = leaf ? 1u : (uint32_t)((a.z >= nrec ? (uint32_t)n : fst[a.z]) - fst[c]);
      if (M || MX) {
        double m, x, y, z;
        if (leaf) {
          const float4 q = rec[c].cm;
          m = (double)q.w;
          x = m * (double)q.x; y = m * (double)q.y; z = m * (double)q.z;
        } else {
          m = mom[c].x; x = mom[c].y; y = mom[c].z; z = mom[c].w;
        }
        if (M) M[k] = m;
        if (MX) { MX[3 * k] = x; MX[3 * k + 1] = y; MX[3 * k + 2] = z; }
      }
    }
    k++;
  }
  if (n_nodes) *n_nodes = k;
  if (k > cap) return fail(ctx, BH_ERR_ARG, "cap %lld < %lld tree nodes", (long long)cap, (long long)k);
  return BH_OK;
}

bh_status bh_get_tree(bh_ctx *ctx, uint8_t *level, uint32_t *first, uint32_t *count, int64_t cap, int64_t *n_nodes) {
  if (!ctx) return BH_ERR_ARG;
  if (!ctx->tree_valid && ctx->steps == 0) return fail(ctx, BH_ERR_STATE, "no tree built yet");
  return export_tree(ctx, level, first, count, nullptr, nullptr, cap, n_nodes);
}

bh_status bh_get_moments(bh_ctx *ctx, double *M, double *MX, int64_t cap) {
  if (!ctx) return BH_ERR_ARG;
  if (!ctx->tree_valid && ctx->steps == 0) return fail(ctx, BH_ERR_STATE, "no tree built yet");
  int64_t nn = 0;
  return export_tree(ctx, nullptr, nullptr, nullptr, M, MX, cap, &nn);
}

bh_status bh_get_quadrupoles(bh_ctx *ctx, double *Q, int64_t cap, int64_t *n_nodes) {
  if (!ctx) return BH_ERR_ARG;
  if (ctx->p.multipole != 2) return fail(ctx, BH_ERR_STATE, "quadrupoles need multipole = 2");
  if (!ctx->tree_valid && ctx->steps == 0) return fail(ctx, BH_ERR_STATE, "no tree built yet");
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = do_sync(ctx);
  if (st) return st;
  const uint32_t nrec = ctx->hstatus->n_records;
  std::vector<Rec> rec(nrec);
  std::vector<double> q((size_t)nrec * 6);
  CK(cudaMemcpy(rec.data(), ctx->W.rec, (size_t)nrec * sizeof(Rec), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(q.data(), ctx->W.qmom, (size_t)nrec * 48, cudaMemcpyDeviceToHost));
  std::vector<uint8_t> lev, leafv;
  st = record_levels(ctx, nrec, lev, leafv);
  if (st) return st;
  int64_t k = 0;
  for (uint32_t c = 0; c < nrec; c++) {
    if (lev[c] > BH_MAXLEVEL) continue;  // bucket member
    if (Q && k < cap)
      for (int j = 0; j < 6; j++) Q[6 * k + j] = leafv[c] ? 0.0 : q[6 * (size_t)c + j];
    k++;
  }
  if (n_nodes) *n_nodes = k;
  if (Q && k > cap) return fail(ctx, BH_ERR_ARG, "cap %lld < %lld tree nodes", (long long)cap, (long long)k);
  return BH_OK;
}

bh_status bh_get_own(bh_ctx *ctx, uint32_t *icount, float *vel, int where) {
  if (!ctx || (where != BH_HOST && where != BH_DEVICE)) return fail(ctx, BH_ERR_ARG, "bad arguments");
  bh_status st = set_dev(ctx);
  if (st) return st;
  const int64_t lo = ctx->own_lo, own_n = ctx->own_hi - ctx->own_lo;
  cudaStream_t s = ctx->stream;
  const cudaMemcpyKind kind = where == BH_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (icount && own_n) CK(cudaMemcpyAsync(icount, ctx->W.icount + lo, (size_t)own_n * 4, kind, s));
  if (vel && own_n) {
    float *dst = where == BH_DEVICE ? vel : ctx->W.accu;
    k_vel4to3<<<blocks_for(own_n), 256, 0, s>>>(dst, ctx->W.vel4, own_n);
    CK(cudaGetLastError());
    if (where == BH_HOST) CK(cudaMemcpyAsync(vel, ctx->W.accu, (size_t)own_n * 12, cudaMemcpyDeviceToHost, s));
  }
  return do_sync(ctx);
}

bh_status bh_get_own_cost(bh_ctx *ctx, uint32_t *trips, int where) {
  if (!ctx || !trips || (where != BH_HOST && where != BH_DEVICE)) return fail(ctx, BH_ERR_ARG, "bad arguments");
  bh_status st = set_dev(ctx);
  if (st) return st;
  const int64_t lo = ctx->own_lo, own_n = ctx->own_hi - ctx->own_lo;
  if (own_n)
    CK(cudaMemcpyAsync(trips, ctx->W.gcost + lo, (size_t)own_n * 4,
                       where == BH_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
  return do_sync(ctx);
}

bh_status bh_set_partition(bh_ctx *ctx, const int64_t *bounds, const float *vel, int where) {
  if (!ctx || !bounds || (where != BH_HOST && where != BH_DEVICE)) return fail(ctx, BH_ERR_ARG, "bad arguments");
  const int P = ctx->p.world, r = ctx->p.rank;
  const int64_t n = ctx->p.n;
  if (bounds[0] != 0 || bounds[P] != n) return fail(ctx, BH_ERR_ARG, "bounds must run from 0 to n");
  for (int k = 0; k < P; k++)
    if (bounds[k + 1] < bounds[k]) return fail(ctx, BH_ERR_ARG, "bounds must not decrease");
  const int64_t lo = bounds[r], hi = bounds[r + 1], own_n = hi - lo;
  if (own_n > ctx->lay.n_own_max)
    return fail(ctx, BH_ERR_ARG, "own range of %lld exceeds the velocity capacity %lld (2x the even share)",
                (long long)own_n, (long long)ctx->lay.n_own_max);
  if (own_n > 0 && !vel) return fail(ctx, BH_ERR_ARG, "velocities of the new own range required");
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = flush_vel(ctx);  // (the new slice's velocities replace them below)
  if (st) return st;
  cudaStream_t s = ctx->stream;
  if (own_n > 0) {
    const float *dv = vel;
    if (where == BH_HOST) {
      CK(cudaMemcpyAsync(ctx->W.accu, vel, (size_t)own_n * 12, cudaMemcpyHostToDevice, s));
      dv = ctx->W.accu;
    }
    k_vel3to4<<<blocks_for(own_n), 256, 0, s>>>(ctx->W.vel4, dv, own_n);
    CK(cudaGetLastError());
  }
  for (int k = 0; k <= P; k++) ctx->bounds[k] = bounds[k];
  ctx->own_lo = lo;
  ctx->own_hi = hi;
  drop_graphs(ctx);  // the walk's target range is baked into the captured steps
  ctx->walked = false;
  return do_sync(ctx);
}

bh_status bh_get_pos4(bh_ctx *ctx, float *pos4, int64_t lo, int64_t hi, int where) {
  if (!ctx || !pos4 || lo < 0 || hi > ctx->p.n || hi < lo || (where != BH_HOST && where != BH_DEVICE))
    return fail(ctx, BH_ERR_ARG, "bad arguments");
  bh_status st = set_dev(ctx);
  if (st) return st;
  if (hi > lo)
    CK(cudaMemcpyAsync(pos4, ctx->W.pos4 + lo, (size_t)(hi - lo) * 16,
                       where == BH_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
  return do_sync(ctx);
}

// ---- the fused exchange (NEXT-1, include/bh.h) -----------------------------
bh_status bh_get_pos4_ptr(bh_ctx *ctx, void **dev_ptr) {
  if (!ctx || !dev_ptr) return fail(ctx, BH_ERR_ARG, "bad arguments");
  *dev_ptr = (void *)ctx->W.pos4;
  return BH_OK;
}

bh_status bh_set_peers(bh_ctx *ctx, void *const *pos4_of_rank) {
  if (!ctx) return BH_ERR_ARG;
  const int P = ctx->p.world, r = ctx->p.rank;
  std::vector<float4 *> peers;
  if (pos4_of_rank) {
    if (P < 2) return fail(ctx, BH_ERR_ARG, "bh_set_peers needs world > 1");
    if (P - 1 > BH_MAX_PEERS) return fail(ctx, BH_ERR_ARG, "world %d exceeds %d peers", P, BH_MAX_PEERS);
    for (int q = 0; q < P; q++) {
      if (q == r) continue;
      if (!pos4_of_rank[q]) return fail(ctx, BH_ERR_ARG, "null replica pointer of rank %d", q);
      if (pos4_of_rank[q] == (void *)ctx->W.pos4) return fail(ctx, BH_ERR_ARG, "rank %d's replica is this rank's", q);
      peers.push_back((float4 *)pos4_of_rank[q]);
    }
  }
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = do_sync(ctx);
  if (st) return st;
  ctx->peers = peers;
  drop_graphs(ctx);  // the replica pointers are baked into the captured steps
  return BH_OK;
}

// one step in two calls, for callers that interleave several ranks' phases
// (bh_step(ctx, 1) == bh_step_phase(ctx, 0) + bh_step_phase(ctx, 1))
bh_status bh_step_phase(bh_ctx *ctx, int phase) {
  if (!ctx || (phase != 0 && phase != 1)) return fail(ctx, BH_ERR_ARG, "bad arguments");
  bh_status st = set_dev(ctx);
  if (st) return st;
  if (phase == 0) {
    st = build_tree(ctx);
    if (st) return st;
    return enqueue_status(ctx);
  }
  if (!ctx->tree_valid) return fail(ctx, BH_ERR_STATE, "bh_step_phase(1) needs bh_step_phase(0) first");
  if (ctx->prof) ctx->prof_calls++;
  const float kick = (float)(ctx->steps == 0 ? 0.5 * ctx->p.dt : ctx->p.dt);
  st = enqueue_walk(ctx, kick);
  if (st) return st;
  ctx->steps++;
  ctx->tree_valid = false;
  return enqueue_status(ctx);
}

bh_status bh_set_pos4(bh_ctx *ctx, const float *pos4, int64_t lo, int64_t hi, int where) {
  if (!ctx || !pos4 || lo < 0 || hi > ctx->p.n || hi < lo || (where != BH_HOST && where != BH_DEVICE))
    return fail(ctx, BH_ERR_ARG, "bad arguments");
  bh_status st = set_dev(ctx);
  if (st) return st;
  if (hi > lo)
    CK(cudaMemcpyAsync(ctx->W.pos4 + lo, pos4, (size_t)(hi - lo) * 16,
                       where == BH_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->tree_valid = false;
  return do_sync(ctx);
}

bh_status bh_get_interactions(bh_ctx *ctx, uint32_t *count, uint64_t *total) {
  if (!ctx) return BH_ERR_ARG;
  bh_status st = set_dev(ctx);
  if (st) return st;
  const int64_t lo = ctx->own_lo, hi = ctx->own_hi, own_n = hi - lo;
  if (count) {
    std::vector<uint32_t> c((size_t)own_n), u((size_t)own_n);
    CK(cudaMemcpyAsync(c.data(), ctx->W.icount + lo, (size_t)own_n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(u.data(), ctx->W.uid + lo, (size_t)own_n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    st = do_sync(ctx);
    if (st) return st;
    for (int64_t k = 0; k < own_n; k++) count[u[k]] = c[k];
  } else {
    st = do_sync(ctx);
    if (st) return st;
  }
  if (total) *total = ctx->hstatus->interactions;
  return BH_OK;
}

bh_status bh_get_stats(bh_ctx *ctx, bh_stats *out) {
  if (!ctx || !out) return BH_ERR_ARG;
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = do_sync(ctx);
  if (st) return st;
  out->n_records = ctx->hstatus->n_records;
  out->n_internal = ctx->hstatus->n_internal;
  out->node_capacity = ctx->lay.cap_rec;
  out->interactions = (int64_t)ctx->hstatus->interactions;
  out->mac_fallbacks = (int64_t)ctx->hstatus->fallbacks;
  out->opens = (int64_t)ctx->hstatus->opens;
  out->record_visits = (int64_t)ctx->hstatus->iters;
  out->leaf_visits = (int64_t)ctx->hstatus->reserved0;
  out->redo_targets = (int64_t)ctx->hstatus->n_redo;
  out->near_sorted = ctx->hstatus->near_ok ? 1 : 0;
  out->sort_bad_keys = ctx->hstatus->n_bad;
  out->interactions_cum = (int64_t)ctx->hstatus->interactions_cum;
  out->opens_cum = (int64_t)ctx->hstatus->opens_cum;
  out->own_begin = ctx->own_lo;
  out->own_end = ctx->own_hi;
  out->steps = ctx->steps;
  return BH_OK;
}

bh_status bh_set_profiling(bh_ctx *ctx, int enable) {
  if (!ctx) return BH_ERR_ARG;
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = do_sync(ctx);
  ctx->prof = enable != 0;
  memset(ctx->prof_ms, 0, sizeof ctx->prof_ms);
  memset(ctx->prof_launches, 0, sizeof ctx->prof_launches);
  ctx->prof_calls = 0;
  return st;
}

bh_status bh_get_profile(bh_ctx *ctx, double *ms, int64_t *launches, int64_t *calls) {
  if (!ctx) return BH_ERR_ARG;
  bh_status st = set_dev(ctx);
  if (st) return st;
  st = do_sync(ctx);
  for (int i = 0; i < BH_NPHASE; i++) {
    if (ms) ms[i] = ctx->prof_ms[i];
    if (launches) launches[i] = ctx->prof_launches[i];
  }
  if (calls) *calls = ctx->prof_calls;
  return st;
}

bh_status bh_set_walk_stats(bh_ctx *ctx, int enable) {
  if (!ctx) return BH_ERR_ARG;
  ctx->walk_stats = enable ? 1 : 0;
  drop_graphs(ctx);  // the captured steps bake in the walk variant
  return BH_OK;
}

bh_status bh_nccl_unique_id(void *id128) {
  if (!id128) return BH_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return BH_ERR_NCCL;
  memcpy(id128, &id, sizeof id);
  return BH_OK;
}

bh_status bh_nccl_comm_init(void **comm, const void *id128, int world, int rank, int device) {
  if (!comm || !id128 || world < 1 || rank < 0 || rank >= world) return BH_ERR_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return BH_ERR_CUDA;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  ncclComm_t c;
  if (ncclCommInitRank(&c, world, id, rank) != ncclSuccess) return BH_ERR_NCCL;
  *comm = (void *)c;
  return BH_OK;
}

bh_status bh_nccl_comm_info(void *comm, int *count, int *rank, int *device) {
  if (!comm) return BH_ERR_ARG;
  ncclComm_t c = (ncclComm_t)comm;
  int v;
  if (count) {
    if (ncclCommCount(c, &v) != ncclSuccess) return BH_ERR_NCCL;
    *count = v;
  }
  if (rank) {
    if (ncclCommUserRank(c, &v) != ncclSuccess) return BH_ERR_NCCL;
    *rank = v;
  }
  if (device) {
    if (ncclCommCuDevice(c, &v) != ncclSuccess) return BH_ERR_NCCL;
    *device = v;
  }
  return BH_OK;
}

bh_status bh_nccl_comm_destroy(void *comm) {
  if (!comm) return BH_OK;
  return ncclCommDestroy((ncclComm_t)comm) == ncclSuccess ? BH_OK : BH_ERR_NCCL;
}

}  // extern "C"
