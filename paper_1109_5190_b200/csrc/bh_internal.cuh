// bh_internal.cuh -- shared definitions of the CUDA path (not part of the ABI).
//
// Data layout in HBM:
//   storage order   : particles are relabelled once, at bh_create, by their
//                     step-0 Morton rank ("storage id" s); rank r of P owns the
//                     contiguous range [own_lo, own_hi).
//   pos4[s]         : float4 (x, y, z, m), replicated on every rank.
//   vel4[s-own_lo]  : float4 (vx, vy, vz, 0), this rank's particles only.
//   uid[s]          : user index of storage id s.
//   sorted arrays   : keys[p] (u64), vals[p] = s, lcp[p] (u8), nstart[p] (u32)
//                     for Morton position p of the current step.
//   walk records    : DFS pre-order array of tree nodes where every particle
//                     has exactly one record (a single-particle leaf, or a
//                     "member" record right after its level-21 bucket):
//                       rec[c].cm  float4 (com32.xyz, M32)       16 B
//                       rec[c].aux uint4  (T_acc, T_rej, skip, drop word) 16 B
//                       (drop word = BH_DROP | c: the walk's resume word of
//                       a target whose MAC test at c was inconclusive)
//                       (one 32-byte sector per record: a lane's visit
//                       touches one sector)
//                     skip(c) = index of the first record after c's subtree,
//                     so DFS next = c + 1 and "accept" jumps to skip(c).
//                     Particle p's records are [nstart[p], nstart[p+1]).
//   level items     : per level 0..22, the records of that level in Morton
//                     order (item_rec, item_clo, lvl_skip, lvl_mom; tree.cu),
//                     so K5 streams each node's children; rec_item[c] maps a
//                     record to its item (fp64 moments of record c = lvl_mom[rec_item[c]]).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bh.h"

#define BH_MAXLEVEL 21
#define BH_NLEVELS 23  // item levels 0 .. 22 (22: bucket members)
#define BH_NPHASE 6
#define BH_MAX_PEERS 15  // bh_set_peers: replicas written by K7 besides the own one (world <= 16)

// the MAC filter's thresholds in the softened domain (com.cu, walk.cu)
#ifndef BH_EPS_FOLD
#define BH_EPS_FOLD 1
#endif

namespace bh {

#define ITEM_LEAF 0x80000000u  // item_rec flag: the item is a particle's own record

// device status block (one per ctx, in the workspace)
enum : uint32_t {
  ERR_NONFINITE_POS = 1u << 0,
  ERR_NONFINITE_FORCE = 1u << 1,
  ERR_NODE_OVERFLOW = 1u << 2,
};

struct DevStatus {
  uint32_t err;
  uint32_t n_records;   // total walk records (nstart[n])
  uint32_t n_internal;
  uint32_t bbox_ticket; // last-block ticket of the bbox reduction
  // per-walk counters (zeroed before every walk; kept contiguous)
  unsigned long long interactions;   // last walk
  unsigned long long fallbacks;      // last walk: fp64 MAC re-evaluations
  unsigned long long opens;          // last walk: MAC tests that opened a node (incl. self leaf)
  unsigned long long iters;          // last stats walk: record loads summed over lanes
  unsigned long long n_redo;         // last walk: targets re-walked with the exact fp64 MAC
  unsigned long long reserved0;      // last stats walk: the record loads of particle records
  uint32_t n_own_groups;             // world > 1: walk groups holding an own particle (walk.cu)
  uint32_t n_long_runs;              // equal-key runs longer than TIE_SHORT queued for k_long_runs (sort.cu)
  uint32_t near_ok;     // this build's sort came from the near-sorted path (sort.cu)
  uint32_t n_bad;       // near-sorted path: keys out of local order, sorted apart
  unsigned long long interactions_cum;  // since create / set_state
  unsigned long long opens_cum;
  float lo[3];
  float L;
  float scale;
  uint32_t pad[3];
  uint32_t lvl_count[24];   // items (records) per level 0..22; [23] = 0
  uint32_t lvl_offset[24];  // exclusive prefix of lvl_count (level-ordered item arrays)
};

struct __align__(32) Rec {
  float4 cm;
  uint4 aux;
};

// record indices (and the sentinel) stay below 2^31: the walk marks a target
// whose fp32 MAC test was inconclusive with resume = BH_DROP | record
#define BH_MAX_RECORDS 0x7ffffffeLL
#define BH_DROP 0x80000000u

// state of a target that dropped out of the fast walk at record cdrop: its
// fp32 partial sums and count over the DFS prefix before cdrop (walk.cu
// k_walk_resume continues the same DFS from there with the exact MAC)
struct __align__(32) ResumeState {
  double ax, ay, az;  // the fast walk's partial sums (fp32 blocks folded in fp64)
  uint32_t cnt;
  uint32_t cdrop;
};

struct Workspace {
  float4 *pos4;
  float4 *vel4;
  uint32_t *uid;
  unsigned long long *keys[2];
  uint32_t *vals[2];
  uint8_t *lcp;
  uint32_t *nstart;   // n + 1
  uint32_t *icount;   // interactions per storage id
  float *accu;        // n * 3, user order (BH_HOST force output staging)
  uint32_t *targets;  // world > 1: the walk groups holding an own particle (walk.cu)
  uint32_t *redo;     // target slots whose fp32 MAC filter was inconclusive
  uint32_t *gcost;      // per storage id: loop trips of its walk group in the last walk (group order)
  double *qmom;       // multipole = 2: per record, fp64 quadrupole xx yy zz xy xz yz (null otherwise)
  float4 *qrec;       // multipole = 2: per record, 2 float4 = fp32 (xx yy zz xy) (xz yz 0 0)
  uint32_t *scan_tmp; // scan tile partials
  uint32_t *sort_hist;    // 8 x 256
  uint32_t *sort_status;  // 8 passes x tiles x 256
  uint32_t *sort_tilectr; // 8
  float *bbox_part;       // partial min/max per block (8 floats)
  Rec *rec;
  ResumeState *resume;  // cap_resume entries (queue slots beyond it re-walk from the root)
  int64_t cap_resume;
  int resume_stack;     // 0: the full resume LIFO; > 0: a smaller one (test hook)
  uint32_t *rec_item;   // per record: its index in the level-ordered item arrays
  float *vstage;        // bh_advance: n x 3 user-order velocities (host upload target)
  // level-ordered items (tree.cu): per level, the records in Morton order
  uint32_t *blkcnt;     // [23][blocks of 256 particles]: item counts, then offsets
  uint32_t *item_rec;   // record index | ITEM_LEAF
  uint32_t *item_clo;   // items of the next level whose first particle precedes this one's
  uint32_t *lvl_skip;   // skip() of the item's record
  double4 *lvl_mom;     // fp64 (M, MX, MY, MZ) of the item
  double *lvl_q;        // multipole = 2: fp64 quadrupole of the item (6 per item; null otherwise)
  float *lvl_rad;       // bounding radius of each item about its com (containment folded into T_acc)
  DevStatus *status;
};

struct Layout {
  int64_t n, cap_rec, cap_int, n_own_max, sort_tiles, scan_tiles, cap_resume, blocks;
  size_t total;
  size_t off[32];
};

// radix sort geometry (sort.cu)
constexpr int SORT_BLOCK = 256;
#ifndef BH_SORT_ITEMS
#define BH_SORT_ITEMS 16
#endif
constexpr int SORT_ITEMS = BH_SORT_ITEMS;
constexpr int SORT_TILE = SORT_BLOCK * SORT_ITEMS;
constexpr int SORT_PASSES = 8;
constexpr int SORT_RADIX = 256;

constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

constexpr int BBOX_BLOCKS = 592;  // 4 x 148 SMs
constexpr int LS_SEG = 1024;      // tree.cu: 256-particle blocks per level-scan segment

Layout make_layout(int64_t n, int world, int64_t node_capacity, int multipole);
void bind_workspace(const Layout &L, void *base, Workspace &W);

// ---- kernel launchers (each returns cudaGetLastError()) -------------------
cudaError_t launch_bbox(const Workspace &W, int64_t n, cudaStream_t s);
cudaError_t launch_keys(const Workspace &W, int64_t n, cudaStream_t s);
cudaError_t launch_keys_prev(const Workspace &W, int64_t n, uint32_t *flags, cudaStream_t s);
cudaError_t launch_sort(const Workspace &W, int64_t n, cudaStream_t s, int *final_buf);
cudaError_t launch_near_sort(const Workspace &W, int64_t n, cudaStream_t s);
cudaError_t launch_sort_bad(const Workspace &W, int64_t tiles, cudaStream_t s);
cudaError_t launch_tie_fixup(const Workspace &W, int64_t n, int buf, cudaStream_t s);
// equal-key runs (reading L13: ties by user index): runs of <= TIE_SHORT keys
// are insertion-sorted by the thread that finds them; longer ones are queued
// (DevStatus.n_long_runs, the list at the start of W.accu) and sorted by
// k_long_runs, one block per run (sort.cu)
constexpr int TIE_SHORT = 32;
__device__ __forceinline__ void tie_run(unsigned long long kp, int64_t p, int64_t n,
                                        const unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals,
                                        const uint32_t *__restrict__ uid, DevStatus *st, uint2 *runs) {
  int64_t e = p + 1;
  while (e + 1 < n && e + 1 - p < TIE_SHORT && keys[e + 1] == kp) ++e;
  if (e + 1 < n && keys[e + 1] == kp) {  // a long run: queue it
    while (e + 1 < n && keys[e + 1] == kp) ++e;
    const uint32_t k = atomicAdd(&st->n_long_runs, 1u);
    runs[k] = make_uint2((uint32_t)p, (uint32_t)(e + 1 - p));
    return;
  }
  for (int64_t i = p + 1; i <= e; ++i) {
    const uint32_t vv = vals[i], u = uid[vv];
    int64_t j = i - 1;
    while (j >= p && uid[vals[j]] > u) { vals[j + 1] = vals[j]; --j; }
    vals[j + 1] = vv;
  }
}
cudaError_t launch_long_runs(const Workspace &W, int64_t n, int buf, cudaStream_t s);
cudaError_t launch_tree(const Workspace &W, int64_t n, int64_t cap_rec, int buf, int cont_fold, cudaStream_t s);
cudaError_t launch_moments(const Workspace &W, int64_t n, double theta, float eps2, int cont_fold, cudaStream_t s,
                           int *launches);
cudaError_t launch_scan_u32(uint32_t *data, int64_t count, uint32_t *tmp, cudaStream_t s);
cudaError_t launch_own_targets(const Workspace &W, int64_t n, int buf, uint32_t own_lo, uint32_t own_hi,
                               cudaStream_t s);

struct WalkArgs {
  int64_t n;            // particles (targets: sorted positions 0 .. n-1)
  int own_check;        // world > 1: walk the P = 1 groups holding an own particle, write own results only
  int buf;              // sort buffer holding vals
  int group;            // walk_group code (66 / 67 / 68: 8 / 4 / 2 lanes per shared traversal)
  int stats;            // 1: also count opened nodes and SIMD slots
  int num_sms;
  int need_cont;        // 0: theta < 1/sqrt(3) and eps > 0 -> no cell containing the
                        //    target can pass the MAC and the self record adds 0
  int mode;             // 0 = forces to acc_out (user order), 1 = fused leapfrog
  float eps2, G;
  float kick, dt;       // mode 1
  double theta2;
  int quad;             // multipole = 2: add each accepted cell's quadrupole field
  uint32_t own_lo, own_hi;
  float *acc_out;       // mode 0: [n][3] device output (may be null)
  int user_order;       // 1: acc_out[uid[s]], 0: acc_out[s - own_lo]
  int n_peers;          // mode 1, bh_set_peers: the other ranks' pos4 replicas K7 also writes
  float4 *const *peer_pos4;
};
cudaError_t launch_walk(const Workspace &W, const WalkArgs &a, cudaStream_t s);
int walk_lanes(int group);

}  // namespace bh
