// sort.cu -- K2: in-house LSD radix sort of (63-bit Morton key, u32 storage id).
//
// PAPER.md:58-60 builds the cube hierarchy with "a recursive algorithm"; on
// B200 the hierarchy is read off the Morton-sorted key array instead, so the
// sort is the tree build's dominant HBM stage.  Reading L13:
// the order is ascending key, ties by ascending user index.
//
// Design (Onesweep, one kernel per 8-bit digit pass, 8 passes):
//   * the 8 digit histograms come for free from K1 (keys.cu);
//   * each CTA takes the next tile (4096 keys) from an atomic ticket, ranks its
//     keys with a warp-level ballot multisplit (stable within the tile),
//     publishes per-digit tile counts and resolves its global offsets by
//     decoupled look-back over earlier tiles (flag + 30-bit count in one
//     32-bit word, so a single relaxed load/store carries both);
//   * keys are reordered in shared memory by digit, then written out, so the
//     stores are runs of consecutive addresses.
// HBM roofline: per pass 12 B read + 12 B written per key -> 192 B/key over 8
// passes.  Stability of LSD radix makes ties follow the input order; a tiny
// fix-up pass re-sorts runs of equal keys by user index (runs are rare: they
// are exact coincidences at the 2^-21 cell size).
#include "bh_internal.cuh"

namespace bh {

constexpr int SORT_WARPS = SORT_BLOCK / 32;
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_PRE = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1;
constexpr int LOOKBACK = 16;  // status words per look-back round trip

struct SortSmem {
  unsigned long long keys[SORT_TILE];
  uint32_t vals[SORT_TILE];
  uint32_t wcount[SORT_WARPS][SORT_RADIX];
  uint32_t dstart[SORT_RADIX];
  int32_t gbase[SORT_RADIX];
  uint32_t scan_tmp[SORT_WARPS * 2];
  uint32_t tile;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// exclusive block scan of one value per thread (SORT_BLOCK threads); returns
// the exclusive prefix, *total receives the block total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *tmp, uint32_t *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < SORT_WARPS ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < SORT_WARPS) tmp[SORT_WARPS + lane] = t;  // inclusive per warp
  }
  __syncthreads();
  uint32_t warp_excl = w ? tmp[SORT_WARPS + w - 1] : 0;
  *total = tmp[2 * SORT_WARPS - 1];
  __syncthreads();
  return warp_excl + x - v;
}

// lanes of the warp whose 8-bit digit equals this lane's, restricted to `act`:
// eight ballots, measured faster here than one match_any per item
__device__ __forceinline__ uint32_t match8(uint32_t act, uint32_t dig) {
  uint32_t peers = act;
#pragma unroll
  for (int b = 0; b < 8; b++) {
    const uint32_t v = __ballot_sync(0xffffffffu, (dig >> b) & 1u);
    peers &= ((dig >> b) & 1u) ? v : ~v;
  }
  return peers;
}

// mode: SORT_FULL runs unless this build's near-sorted path succeeded
// (st->near_ok); SORT_BAD sorts the near-sorted path's st->n_bad out-of-order
// keys and runs only if that path is still on.
enum { SORT_FULL = 0, SORT_BAD = 1 };
#ifndef BH_SORT_PERSIST
#define BH_SORT_PERSIST 1
#endif
constexpr int64_t SORT_PERSIST_GRID = 2 * 148;  // 2 CTAs per SM (__launch_bounds__ below)

__global__ void __launch_bounds__(SORT_BLOCK, 2) k_onesweep(const unsigned long long *__restrict__ kin,
                                                         const uint32_t *__restrict__ vin,
                                                         unsigned long long *__restrict__ kout,
                                                         uint32_t *__restrict__ vout, int64_t n_arg, int shift,
                                                         const uint32_t *__restrict__ hist, uint32_t *status,
                                                         uint32_t *tile_ctr, const DevStatus *__restrict__ st,
                                                         int mode) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem &S = *reinterpret_cast<SortSmem *>(smem_raw);
  const uint32_t near = st->near_ok;
  if (mode == SORT_FULL ? near != 0u : near == 0u) return;  // uniform
  const int64_t n = mode == SORT_FULL ? n_arg : (int64_t)st->n_bad;
  // exactly the blocks the data needs take a tile ticket (tickets 0 .. need-1
  // all go out); the rest of a capacity-sized grid (SORT_BAD) leaves at once
  const int64_t need = n > 0 ? (n + SORT_TILE - 1) / SORT_TILE : 1;
  if ((int64_t)blockIdx.x >= need) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // BH_SORT_PERSIST: a grid of at most 2 CTAs per SM, each taking tickets
  // until they run out (tiles in ticket order, so the look-back only waits on
  // tiles that running CTAs hold); a pass that does not run -- the full path
  // of a near-sorted build, the bad-key path's capacity tail -- costs ~300
  // CTAs that leave at once instead of one per tile
  for (;;) {
  if (tid == 0) S.tile = atomicAdd(tile_ctr, 1u);
  for (int i = tid; i < SORT_WARPS * SORT_RADIX; i += SORT_BLOCK) (&S.wcount[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = S.tile;
  if ((int64_t)tile >= need) break;  // every ticket has gone out
  const int64_t tbase = (int64_t)tile * SORT_TILE;
  if (tbase >= n && tile > 0) break;  // past the data (SORT_BAD sizes its grid for the capacity)
  const int64_t wbase = tbase + (int64_t)warp * 32 * SORT_ITEMS;

  unsigned long long k[SORT_ITEMS];
  uint32_t v[SORT_ITEMS], rank[SORT_ITEMS];
#pragma unroll
  for (int j = 0; j < SORT_ITEMS; j++) {
    int64_t idx = wbase + j * 32 + lane;
    k[j] = idx < n ? kin[idx] : 0ull;
    // the first pass has no payload array: the payload is the storage id itself
    v[j] = vin ? (idx < n ? vin[idx] : 0u) : (uint32_t)idx;
  }
  // warp multisplit ranking, stable in (j, lane) order
#pragma unroll
  for (int j = 0; j < SORT_ITEMS; j++) {
    int64_t idx = wbase + j * 32 + lane;
    bool valid = idx < n;
    uint32_t act = __ballot_sync(0xffffffffu, valid);
    const uint32_t peers_j = match8(act, (uint32_t)(k[j] >> shift) & 0xffu);
    if (valid) {
      uint32_t dig = (uint32_t)(k[j] >> shift) & 0xffu;
      uint32_t peers = peers_j;
      int leader = 31 - __clz(peers);
      uint32_t below = __popc(peers & lanemask_lt());
      uint32_t base = 0;
      if (lane == leader) {
        base = S.wcount[warp][dig];
        S.wcount[warp][dig] = base + __popc(peers);
      }
      base = __shfl_sync(act, base, leader);
      rank[j] = base + below;
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit (thread == digit): exclusive offsets across warps, tile total
  const int dd = tid;
  uint32_t tot = 0;
#pragma unroll
  for (int w = 0; w < SORT_WARPS; w++) {
    uint32_t c = S.wcount[w][dd];
    S.wcount[w][dd] = tot;
    tot += c;
  }
  uint32_t dummy;
  uint32_t dstart = block_excl_scan(tot, S.scan_tmp, &dummy);
  uint32_t gdig = block_excl_scan(hist[dd], S.scan_tmp, &dummy);
  S.dstart[dd] = dstart;
  // decoupled look-back for digit dd
  uint32_t *my = status + (size_t)tile * SORT_RADIX + dd;
  uint32_t excl = 0;
  if (tile == 0) {
    st_relaxed(my, FLAG_PRE | tot);
  } else {
    st_relaxed(my, FLAG_AGG | tot);
    // look back LB tiles per round trip: the nearest inclusive prefix is
    // usually a whole wave of resident tiles back, so one status word per
    // round trip would serialise the pass on load latency
    int64_t t = (int64_t)tile - 1;
    for (;;) {
      uint32_t sv[LOOKBACK];
#pragma unroll
      for (int i = 0; i < LOOKBACK; i++)
        sv[i] = t - i >= 0 ? ld_relaxed(status + (size_t)(t - i) * SORT_RADIX + dd) : FLAG_PRE;
      int used = 0;
      bool done = false;
#pragma unroll
      for (int i = 0; i < LOOKBACK; i++) {
        if (done || used < i) continue;  // stopped at an unpublished word
        const uint32_t f = sv[i] & ~VAL_MASK;
        if (f == 0) continue;
        excl += sv[i] & VAL_MASK;
        used = i + 1;
        done = f == FLAG_PRE;
      }
      if (done) break;
      t -= used;
    }
    st_relaxed(my, FLAG_PRE | (excl + tot));
  }
  S.gbase[dd] = (int32_t)(gdig + excl) - (int32_t)dstart;
  __syncthreads();
  // scatter into shared memory in tile-sorted order
#pragma unroll
  for (int j = 0; j < SORT_ITEMS; j++) {
    int64_t idx = wbase + j * 32 + lane;
    if (idx < n) {
      uint32_t dig = (uint32_t)(k[j] >> shift) & 0xffu;
      uint32_t loc = S.dstart[dig] + S.wcount[warp][dig] + rank[j];
      S.keys[loc] = k[j];
      S.vals[loc] = v[j];
    }
  }
  __syncthreads();
  int64_t rem = n - tbase;
  const int valid_n = rem < SORT_TILE ? (int)rem : SORT_TILE;
  for (int i = tid; i < valid_n; i += SORT_BLOCK) {
    unsigned long long key = S.keys[i];
    uint32_t dig = (uint32_t)(key >> shift) & 0xffu;
    int64_t g = (int64_t)S.gbase[dig] + i;
    kout[g] = key;
    vout[g] = S.vals[i];
  }
  if (!BH_SORT_PERSIST) break;
  __syncthreads();  // S is reused by the next tile
  }
}

// ties: re-sort each run of equal keys by user index (reading L13): short
// runs in place by the thread that finds them, long ones by k_long_runs.
__global__ void k_tie_fixup(const unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals,
                            const uint32_t *__restrict__ uid, int64_t n, DevStatus *st, uint2 *runs) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p + 1 >= n) return;
  unsigned long long kp = keys[p];
  if (keys[p + 1] != kp) return;
  if (p > 0 && keys[p - 1] == kp) return;
  tie_run(kp, p, n, keys, vals, uid, st, runs);
}

// One block per queued long run [p, p + k): order vals by uid[vals] (the user
// indices are distinct).  Tiles of LR_TILE are bitonic-sorted in shared memory;
// runs longer than a tile are then merged pairwise by rank (an element's place
// in the merged run = its place in its own sorted part + the count of the other
// part's smaller keys), ping-ponging between (uid, val) pairs in scratch and
// vals itself (keys re-gathered from uid).  Never on the path of ordinary
// inputs (runs need many particles in one level-21 cell); bounded work
// O(k log k) where a single-thread insertion sort was O(k^2).
constexpr int LR_TILE = 4096;
__global__ void __launch_bounds__(512) k_long_runs(uint32_t *__restrict__ vals, const uint32_t *__restrict__ uid,
                                                   const DevStatus *__restrict__ st, const uint2 *__restrict__ runs,
                                                   uint2 *__restrict__ scratch) {
  __shared__ uint32_t sk[LR_TILE], sv[LR_TILE];
  const uint32_t nr = st->n_long_runs;
  for (uint32_t r = blockIdx.x; r < nr; r += gridDim.x) {
    const uint2 run = runs[r];
    const uint32_t p = run.x, k = run.y;
    uint32_t *v = vals + p;
    uint2 *sc = scratch + p;  // this run's merge slots
    // 1) sort each tile in shared memory
    for (uint32_t t0 = 0; t0 < k; t0 += LR_TILE) {
      const uint32_t len = min((uint32_t)LR_TILE, k - t0);
      for (uint32_t i = threadIdx.x; i < LR_TILE; i += blockDim.x) {
        const uint32_t vv = i < len ? v[t0 + i] : 0xffffffffu;
        sk[i] = i < len ? uid[vv] : 0xffffffffu;
        sv[i] = vv;
      }
      __syncthreads();
      for (uint32_t size = 2; size <= LR_TILE; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
          for (uint32_t i = threadIdx.x; i < LR_TILE; i += blockDim.x) {
            const uint32_t j = i ^ stride;
            if (j > i) {
              const bool up = (i & size) == 0;
              const uint32_t a = sk[i], b = sk[j];
              if ((a > b) == up) {
                sk[i] = b; sk[j] = a;
                const uint32_t t = sv[i]; sv[i] = sv[j]; sv[j] = t;
              }
            }
          }
          __syncthreads();
        }
      }
      for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) {
        if (k <= (uint32_t)LR_TILE) v[t0 + i] = sv[i];
        else sc[t0 + i] = make_uint2(sk[i], sv[i]);
      }
      __syncthreads();
    }
    if (k <= (uint32_t)LR_TILE) continue;
    // 2) merge sorted parts of width w pairwise: scratch -> vals -> scratch ...
    bool in_scratch = true;
    for (uint32_t w = LR_TILE; w < k; w <<= 1) {
      for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        const uint32_t base = i / (2 * w) * (2 * w);
        const bool left = i - base < w;
        const uint32_t lo = left ? base + w : base;  // the other part
        const uint32_t hi = left ? min(base + 2 * w, k) : base + w;
        const uint32_t key = in_scratch ? sc[i].x : uid[v[i]];
        const uint32_t val = in_scratch ? sc[i].y : v[i];
        uint32_t a = lo, b = hi;  // count of the other part's keys < key
        while (a < b) {
          const uint32_t m = (a + b) >> 1;
          const uint32_t km = in_scratch ? sc[m].x : uid[v[m]];
          if (km < key) a = m + 1; else b = m;
        }
        const uint32_t pos = base + (left ? i - base : i - base - w) + (a - lo);
        if (hi <= lo) {  // a left part without a right partner stays in place
          if (in_scratch) v[i] = val; else sc[i] = make_uint2(key, val);
        } else if (in_scratch) {
          v[pos] = val;
        } else {
          sc[pos] = make_uint2(key, val);
        }
      }
      __syncthreads();
      in_scratch = !in_scratch;
    }
    if (in_scratch)
      for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) v[i] = sc[i].y;
    __syncthreads();
  }
}

cudaError_t launch_sort(const Workspace &W, int64_t n, cudaStream_t s, int *final_buf) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int64_t tiles = (n + SORT_TILE - 1) / SORT_TILE;
  const int64_t grid = BH_SORT_PERSIST && tiles > SORT_PERSIST_GRID ? SORT_PERSIST_GRID : tiles;
  int src = 0;
  for (int pass = 0; pass < SORT_PASSES; pass++) {
    k_onesweep<<<(unsigned)grid, SORT_BLOCK, sizeof(SortSmem), s>>>(
        W.keys[src], pass == 0 ? nullptr : W.vals[src], W.keys[src ^ 1], W.vals[src ^ 1], n, 8 * pass, W.sort_hist + pass * SORT_RADIX,
        W.sort_status + (size_t)pass * tiles * SORT_RADIX, W.sort_tilectr + pass, W.status, SORT_FULL);
    src ^= 1;
  }
  *final_buf = src;
  return cudaGetLastError();
}

// the near-sorted path's bad keys: keys[1][0 .. st->n_bad) with their ids, 8
// passes through keys[0] and back (the count lives on the device; the grid is
// sized for the capacity, tiles past the data return at once)
cudaError_t launch_sort_bad(const Workspace &W, int64_t tiles, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t grid = BH_SORT_PERSIST && tiles > SORT_PERSIST_GRID ? SORT_PERSIST_GRID : tiles;
  int src = 1;
  for (int pass = 0; pass < SORT_PASSES; pass++) {
    k_onesweep<<<(unsigned)grid, SORT_BLOCK, sizeof(SortSmem), s>>>(
        W.keys[src], W.vals[src], W.keys[src ^ 1], W.vals[src ^ 1], 0, 8 * pass, W.sort_hist + pass * SORT_RADIX,
        W.sort_status + (size_t)pass * tiles * SORT_RADIX, W.sort_tilectr + pass, W.status, SORT_BAD);
    src ^= 1;
  }
  return cudaGetLastError();
}

// scratch layout in W.accu (12 n bytes, free during the build): the list of
// long runs (at most n / (TIE_SHORT + 1) uint2) at the front, then n uint2
// merge slots indexed by sorted position (8 n bytes: 8 n + 8 n / 33 < 12 n)
static uint2 *long_run_list(const Workspace &W) { return (uint2 *)W.accu; }
static uint2 *long_run_scratch(const Workspace &W, int64_t n) {
  return (uint2 *)W.accu + (n / (TIE_SHORT + 1) + 2);
}

cudaError_t launch_long_runs(const Workspace &W, int64_t n, int buf, cudaStream_t s) {
  if (n < TIE_SHORT + 1) return cudaSuccess;
  k_long_runs<<<148, 512, 0, s>>>(W.vals[buf], W.uid, W.status, long_run_list(W), long_run_scratch(W, n));
  return cudaGetLastError();
}

cudaError_t launch_tie_fixup(const Workspace &W, int64_t n, int buf, cudaStream_t s) {
  if (n < 2) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(&W.status->n_long_runs, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  k_tie_fixup<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(W.keys[buf], W.vals[buf], W.uid, n, W.status,
                                                           long_run_list(W));
  return launch_long_runs(W, n, buf, s);
}

}  // namespace bh
