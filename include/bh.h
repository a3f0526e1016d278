/*
 * bh.h -- C ABI of libbh.so, the B200 (sm_100a) Barnes-Hut step.
 *
 * The library computes, per time step, the paper's data-parallel hot path
 * (arxiv 1109.5190, PAPER.md):
 *   - the adaptive octree, "cubes subdivided until there is one particle per
 *     sub-cube" (§1), built from 63-bit Morton keys;
 *   - "center of mass ... of each of the cubes";
 *   - the force stage, "the most computationally intensive part"
 *     (§3), with the criterion "treated as a single body only
 *     if D is greater than r/theta" (Fig. 1);
 *   - "compute the next iteration values" (Fig. 2c): a
 *     kick-drift leapfrog.
 * DESIGN.md §3 lists the readings where the paper is silent (L1-L24: r is the
 * cell side, D is measured to the centre of mass, the test is strict, cells
 * containing the target are always opened, Plummer softening, 21-level cap with
 * buckets, ties sort by user index, fp64 moments in child order).
 *
 * Conventions for every entry point:
 *   - Return a bh_status; BH_OK == 0.  bh_last_error(ctx) gives text.
 *   - `where` says where caller pointers live: BH_HOST (pageable or pinned host
 *     memory) or BH_DEVICE (device pointers on the ctx's device, e.g. a torch
 *     tensor's data_ptr()).
 *   - Caller arrays are only borrowed for the duration of the call.  Inputs are
 *     copied in, outputs are written into caller buffers.
 *   - Layouts: mass float[n]; pos, vel, acc float[n][3] row-major (x,y,z per
 *     particle); all in USER order (the caller's particle index) unless noted.
 *   - All device memory is carved out of the caller's `workspace`
 *     (bh_workspace_bytes); the library never calls cudaMalloc.  The workspace
 *     must stay allocated until bh_destroy.  Besides it the library owns only a
 *     few hundred bytes of pinned host status memory, CUDA events and (once
 *     bh_advance is called) a second stream for its velocity upload.
 *   - All device work is enqueued on params.stream (NULL: a library-owned
 *     non-blocking stream); bh_advance's upload stream is joined to it by an
 *     event and drained before bh_advance returns.  bh_build_tree, bh_compute_forces with a device
 *     output and bh_step are asynchronous; errors found on the device (non-finite
 *     positions, infinite forces, node-capacity overflow) are reported by the
 *     next synchronising call: bh_sync, any getter, a BH_HOST output, or the next
 *     bh_step once the previous one has completed.
 *   - A ctx is not thread-safe; use one ctx per device / rank.
 */
#ifndef BH_H
#define BH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bh_ctx bh_ctx; /* opaque; one per rank / device */

typedef enum {
    BH_OK = 0,
    BH_ERR_ARG = -1,       /* invalid argument; nothing was changed            */
    BH_ERR_CUDA = -2,      /* a CUDA runtime call or kernel launch failed       */
    BH_ERR_OOM = -3,       /* workspace too small or tree node capacity exceeded */
    BH_ERR_STATE = -4,     /* call out of order (e.g. forces before a tree)     */
    BH_ERR_NONFINITE = -5, /* NaN/Inf position, or eps == 0 with r == 0         */
    BH_ERR_NCCL = -6       /* an NCCL call failed                               */
} bh_status;

enum { BH_HOST = 0, BH_DEVICE = 1 };

typedef struct {
    int64_t n;          /* particle count, 1 <= n <= 2^30 ("n particles")   */
    double theta;       /* opening angle >= 0; 0 = never accept a cell    */
    double eps;         /* Plummer softening >= 0 (reading L6)                               */
    double G;           /* gravitational constant > 0 (reading L7; applied as a final scale) */
    double dt;          /* time step > 0 (reading L8)                                       */
    int device;         /* CUDA device ordinal                                               */
    int rank, world;    /* Morton-range shard `rank` of `world` ranks (world == 1: one GPU) */
    void *stream;       /* cudaStream_t for all work; NULL = library-owned stream            */
    void *nccl_comm;    /* ncclComm_t over the `world` ranks, or NULL (see bh_step)          */
    void *workspace;    /* device memory of >= bh_workspace_bytes(params) bytes, 256-aligned */
    size_t workspace_bytes;
    int64_t node_capacity; /* tree records (internal nodes + particles); 0 = default
                              (n + max(n, min(21 n, 2^22)) + 64, which always fits
                              n <= 199,728 and typical inputs above that)              */
    int walk_group;     /* force-walk group shape: 0 = automatic (code 68 below 2^19 particles;
                           69 up to 2^22 and for theta < 0.6 above; 70 for theta >= 0.6 from
                           2^22; with multipole = 2: 67 for theta < 0.6 from 2^22, else 68);
                           66 / 67 / 68 = 8 / 4 / 2 lanes x 2 targets share one traversal,
                           69 / 70 = 2 / 1 lanes x 4 targets.  Interaction counts never depend
                           on it; the fp32 block sums of a target follow its group's walk, so
                           forces agree to rounding across codes and bitwise for one code at
                           any rank count                                                    */
    int multipole;      /* cell expansion: 0 or 1 = monopole (the paper's method); 2 = monopole
                           + traceless quadrupole about the cell's centre of mass (the paper's
                           future work; reading L25 of DESIGN.md §3).  The MAC
                           and the interaction counts do not change                         */
} bh_params;

/* Bytes of device workspace the ctx needs for these params (n, world,
 * node_capacity are read).  Returns 0 if the params are invalid. */
size_t bh_workspace_bytes(const bh_params *p);

/* Create a ctx and load the initial state (mass[n], pos[n][3], vel[n][3] or
 * NULL for zero velocities), all in user order, from `where`.  Every rank
 * passes the FULL state.  Computes the step-0 Morton order, which fixes the
 * storage order and (world > 1) each rank's owned contiguous Morton range.
 * Synchronises the stream. */
bh_status bh_create(bh_ctx **out, const bh_params *p, const float *mass, const float *pos,
                    const float *vel, int where);

/* Replace the state (user order; vel may be NULL = zero; mass may be NULL =
 * keep the current masses, so a caller that only moves particles sends 24 B per
 * particle).  Keeps the storage order of bh_create and resets the step counter
 * (the next bh_step applies the half kick, reading L8).  Asynchronous for
 * BH_DEVICE inputs. */
bh_status bh_set_state(bh_ctx *ctx, const float *mass, const float *pos, const float *vel, int where);

/* K0-K5: root cube, Morton keys, radix sort, octree, mass / centre of mass on
 * the current positions.  Asynchronous. */
bh_status bh_build_tree(bh_ctx *ctx);

/* K6: accelerations a_i = G sum m_s (x_s - x_i) / (|x_s - x_i|^2 + eps^2)^(3/2)
 * over each particle's Barnes-Hut frontier, for this rank's particles, written
 * to acc[n][3] in user order (entries of other ranks' particles untouched).
 * acc may be NULL (only interaction counts are produced).  Needs
 * bh_build_tree first (BH_ERR_STATE otherwise).  Synchronises for BH_HOST. */
bh_status bh_compute_forces(bh_ctx *ctx, float *acc, int where);

/* nsteps x (K0-K5 tree, K6+K7 walk fused with the leapfrog kick-drift on this
 * rank's particles, K8 exchange of the updated positions).  Step k == 0 of the
 * ctx applies v += a dt/2, later steps v += a dt, then x += v dt, so after
 * k >= 1 steps velocities are the staggered v_{k-1/2}.  With world > 1 the
 * exchange is a grouped ncclBroadcast of every rank's slice over nccl_comm;
 * with nccl_comm == NULL the exchange is skipped (single-GPU rank emulation:
 * only this rank's slice advances).  Asynchronous. */
bh_status bh_step(bh_ctx *ctx, int nsteps);

/* bh_set_state(mass, pos, vel, where) + bh_step(nsteps) + bh_get_state(pos_out,
 * vel_out, where) in one call, for callers that keep the state on the host:
 * the velocities (read only by the first walk's leapfrog) are uploaded on a
 * second stream while the first tree is built, after the positions.  mass NULL
 * keeps the masses, vel NULL means zero velocities, pos_out / vel_out NULL skip
 * that output.  Synchronous: every buffer is borrowed only for the call.
 * Results are identical to the three calls. */
bh_status bh_advance(bh_ctx *ctx, const float *mass, const float *pos, const float *vel, int nsteps, float *pos_out,
                     float *vel_out, int where);

/* Wait for all enqueued work; report device-side errors. */
bh_status bh_sync(bh_ctx *ctx);

/* Free the ctx (not the workspace).  NULL is a no-op. */
bh_status bh_destroy(bh_ctx *ctx);

/* ---- inspection (synchronising; user order unless noted) ---------------- */

/* Positions of all particles and velocities (staggered, see bh_step) of this
 * rank's particles; either pointer may be NULL. */
bh_status bh_get_state(bh_ctx *ctx, float *pos, float *vel, int where);

/* Root cube of the last tree: lo[3], side L and quantisation scale 2^21/L. */
bh_status bh_get_root(bh_ctx *ctx, float *lo3, float *L, float *scale);

/* Sorted 63-bit keys (Morton order) and perm[s] = user index of sorted slot s
 * (ties by ascending user index).  Host pointers, n entries each. */
bh_status bh_get_keys(bh_ctx *ctx, uint64_t *keys, uint32_t *perm);

/* Octree in DFS pre-order (children in Morton digit order): level, first
 * sorted particle, particle count per node, for internal nodes, level-21
 * buckets and single-particle leaves (not bucket members).  Host pointers of
 * `cap` entries (any may be NULL); *n_nodes receives the node count; returns
 * BH_ERR_ARG if cap is too small (n_nodes still set). */
bh_status bh_get_tree(bh_ctx *ctx, uint8_t *level, uint32_t *first, uint32_t *count,
                      int64_t cap, int64_t *n_nodes);

/* fp64 mass M and first moment MX[3] (com = MX / M) of the nodes of
 * bh_get_tree, same order; host pointers of `cap` entries. */
bh_status bh_get_moments(bh_ctx *ctx, double *M, double *MX, int64_t cap);

/* Interactions of the last force walk (accepted cells + particles j != i,
 * reading L21) per particle in user order (this rank's particles; NULL ok) and
 * summed over this rank (NULL ok). */
bh_status bh_get_interactions(bh_ctx *ctx, uint32_t *count, uint64_t *total);

/* Ownership (multi-GPU load balance; the paper's dynamic
 * load-balancing theme).  Rank r owns the storage ids
 * [bounds[r], bounds[r+1]) (storage id = the particle's step-0 Morton rank);
 * bh_create starts from the even split n r / P.
 * bh_get_own: this rank's own slice in storage order -- icount[own] (the last
 *   walk's per-particle interactions, a cost estimate; NULL ok) and vel[own][3]
 *   (the staggered velocities; NULL ok).  where = BH_HOST / BH_DEVICE.  Syncs.
 * bh_set_partition: new bounds[world + 1] (identical on every rank; 0 = bounds[0]
 *   <= ... <= bounds[world] = n) and the velocities of the new own slice
 *   vel[bounds[r+1] - bounds[r]][3] in storage order (gathered by the caller,
 *   e.g. paper_1109_5190_b200.dist.rebalance).  The own range may hold at most
 *   2 ceil(n / P) + 1 particles (BH_ERR_ARG otherwise).  Positions are
 *   replicated and unaffected; results do not depend on the partition.  Syncs. */
bh_status bh_get_own(bh_ctx *ctx, uint32_t *icount, float *vel, int where);

/* bh_get_own_cost: trips[own] = the loop trips of the walk group each own
 * particle was last walked in (storage order, uint32[own_hi - own_lo]; 0
 * before the first walk) -- a walk-TIME cost estimate: a rank's walk time
 * follows the summed trips of its groups more closely than their interaction
 * counts.  Ownership-balancing input for bh_set_partition.
 * where = BH_HOST / BH_DEVICE.  Syncs. */
bh_status bh_get_own_cost(bh_ctx *ctx, uint32_t *trips, int where);

/* multipole = 2: the fp64 quadrupoles of the tree nodes in bh_get_tree's order,
 * Q[node][6] = (xx, yy, zz, xy, xz, yz) about the node's centre of mass
 * (particles: 0).  Q may be NULL to query *n_nodes.  Syncs. */
bh_status bh_get_quadrupoles(bh_ctx *ctx, double *Q, int64_t cap, int64_t *n_nodes);

/* The replicated positions as the exchange moves them: pos4[k] = (x, y, z, m)
 * of storage id lo + k, k < hi - lo (storage order, float[hi-lo][4]).  With no
 * NCCL communicator (nccl_comm = NULL) bh_step skips K8, and a caller can run
 * its own exchange (MPI, host, or -- in tests/test_gpu_parity.py -- several
 * single-GPU ranks in one process): after every step, copy each owner's
 * [bounds[r], bounds[r+1]) slice into every other rank.  bh_set_pos4
 * invalidates the tree.  Both sync. */
bh_status bh_get_pos4(bh_ctx *ctx, float *pos4, int64_t lo, int64_t hi, int where);
bh_status bh_set_pos4(bh_ctx *ctx, const float *pos4, int64_t lo, int64_t hi, int where);
bh_status bh_set_partition(bh_ctx *ctx, const int64_t *bounds, const float *vel, int where);

/* The fused exchange (the per-iteration global barrier
 * of PAPER.md:441-444, §3).  K8 is folded into K7: the walk's leapfrog epilogue
 * stores each updated own position into this rank's pos4 AND into every other
 * rank's replica (peer memory: NVLink stores, 16 B per particle per peer), so
 * the exchange overlaps the walk instead of following it.
 * bh_get_pos4_ptr: the device address of this ctx's pos4 replica (float4[n],
 *   storage order, inside the caller's workspace: same offset on every rank),
 *   for the caller to share (same process: the pointer; other processes: a CUDA
 *   IPC handle of the workspace, paper_1109_5190_b200.dist.share_replicas).
 * bh_set_peers: pos4_of_rank[world] = every rank's replica as a device pointer
 *   valid on this ctx's device (this rank's own entry is ignored); NULL turns
 *   the fused exchange off (back to K8's grouped ncclBroadcast).  The pointers
 *   are borrowed until the next bh_set_peers / bh_destroy; world - 1 <= 15.
 *   Ordering: with an NCCL communicator every step runs build -> barrier (a
 *   one-word ncclAllReduce) -> walk with peer stores -> barrier, captured in
 *   the step graph.  Without one, the caller orders the ranks' phases with
 *   bh_step_phase (all ranks' phase 0, then all ranks' phase 1) and a device
 *   sync between them; bh_step / bh_advance then return BH_ERR_STATE (nothing
 *   would order this rank's stores after the others' builds).  Results are
 *   bitwise those of bh_step with the
 *   broadcast (tests/test_gpu_parity.py, tests/test_gpu_multiproc.py).  Syncs.
 * bh_step_phase: one step in two calls; phase 0 = K0-K5 (the tree of the
 *   current positions), phase 1 = K6-K8 (walk, leapfrog, exchange);
 *   bh_step(ctx, 1) == phase 0 + phase 1.  BH_ERR_STATE for phase 1 without a
 *   fresh phase 0.  Direct launches (no graph).  Asynchronous. */
bh_status bh_get_pos4_ptr(bh_ctx *ctx, void **dev_ptr);
bh_status bh_set_peers(bh_ctx *ctx, void *const *pos4_of_rank);
bh_status bh_step_phase(bh_ctx *ctx, int phase);

typedef struct {
    int64_t n_records;      /* walk records: tree nodes + bucket members          */
    int64_t n_internal;     /* internal nodes incl. buckets                       */
    int64_t node_capacity;  /* capacity in records                                */
    int64_t interactions;   /* last walk, this rank                               */
    int64_t mac_fallbacks;  /* last walk: fp32 MAC filter inconclusive -> fp64    */
    int64_t own_begin, own_end; /* this rank's range of storage indices          */
    int64_t steps;          /* steps taken since create / set_state              */
    int64_t opens;          /* last walk: MAC tests that opened a node             */
    int64_t interactions_cum; /* all walks since bh_create                        */
    int64_t opens_cum;
    int64_t record_visits;  /* last stats walk (bh_set_walk_stats): record loads, per lane */
    int64_t redo_targets;   /* last walk: targets whose fp32 MAC test was inconclusive,
                               continued with the exact fp64 test (k_walk_resume)        */
    int64_t near_sorted;    /* last build: 1 if the sort took the near-sorted path (keys
                               in the previous build's order, out-of-order keys sorted
                               apart and merged), 0 if the full radix sort ran           */
    int64_t sort_bad_keys;  /* last build, near-sorted path: keys out of local order     */
    int64_t leaf_visits;    /* last stats walk: the record loads of particle records     */
} bh_stats;
bh_status bh_get_stats(bh_ctx *ctx, bh_stats *out);

/* Per-phase device time (CUDA events on the ctx stream), accumulated over the
 * calls made while profiling is on.  Phases: 0 bbox (root cube), 1 keys + sort,
 * 2 tree, 3 moments, 4 walk(+integrate), 5 exchange.  ms[6], launches[6]. */
bh_status bh_set_profiling(bh_ctx *ctx, int enable);
bh_status bh_get_profile(bh_ctx *ctx, double *ms, int64_t *launches, int64_t *calls);

/* Walk statistics (the opens of bh_get_stats: MAC tests that opened a node)
 * cost a few instructions per visited node; they are off by default
 * (interactions are always counted). */
bh_status bh_set_walk_stats(bh_ctx *ctx, int enable);

const char *bh_last_error(const bh_ctx *ctx);
const char *bh_status_string(int status);

/* ---- NCCL bootstrap (world > 1) ----------------------------------------- */
/* 128-byte ncclUniqueId generated on one rank and shared by the caller
 * (e.g. a torch.distributed broadcast). */
bh_status bh_nccl_unique_id(void *id128);
bh_status bh_nccl_comm_init(void **comm, const void *id128, int world, int rank, int device);
/* The communicator's rank count, this rank and its CUDA device
 * (ncclCommCount / ncclCommUserRank / ncclCommCuDevice; NULL outputs skipped).
 * bench.py logs them so a run shows how many ranks NCCL actually spans. */
bh_status bh_nccl_comm_info(void *comm, int *count, int *rank, int *device);
bh_status bh_nccl_comm_destroy(void *comm);

#ifdef __cplusplus
}
#endif
#endif /* BH_H */
