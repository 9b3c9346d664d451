// K2: tile binning.
//
//   1. stable radix sort of the N Gaussians by depth (float64 bits of t_z,
//      the reference's exact key; ties keep ascending cloud index) -> order[]
//   2. exclusive scan of tiles-touched in depth order -> entry offsets, E
//   3. duplicate: Gaussian order[s] writes one (tile, id) entry per covered
//      tile at offsets[s]; entries are therefore in (depth, index) order
//   4. stable radix sort of the entries by tile id over ceil(log2 T) bits
//      -> entry_splat[] sorted by (tile, depth, index) = np.lexsort((row,
//      depth, tile)) of frontend.py:169
//   5. tile ranges by binary search (= np.searchsorted, frontend.py:171-173)
//
// Sorting the N Gaussians once (64-bit keys, L2-resident) and then only the
// ~10 tile bits of the E entries replaces a 74-bit (tile|depth64) sort of E
// keys: two passes over E instead of ten.
#include <limits.h>
#include <stdlib.h>
#include <string.h>

#include "xg_sort.cuh"

namespace xg {
namespace {

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

__global__ void k_iota(uint32_t* v, long long n, uint32_t* n_dev) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
  if (i == 0) *n_dev = (uint32_t)n;
}

// One warp per 32 consecutive depth-sorted Gaussians.  Their entries are
// contiguous ([offsets[s0], offsets[s0] + total)), so the warp writes them
// cooperatively - lane e of each round writes entry base + e - which keeps
// every store coalesced regardless of how many tiles each Gaussian covers.
__global__ void k_duplicate(const uint32_t* __restrict__ order, const uint32_t* __restrict__ n_tiles,
                            const ushort4* __restrict__ rect, const uint32_t* __restrict__ offsets,
                            long long n, int ntx, long long cap, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals, uint32_t* counters) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  uint32_t g = 0, cnt = 0;
  ushort4 r = make_ushort4(0, 0, 0, 0);
  long long off = 0;
  if (s < n) {
    g = order[s];
    cnt = n_tiles[g];
    off = offsets[s];
    if (cnt) r = rect[g];
  }
  // inclusive warp scan of the counts
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  const uint32_t excl = incl - cnt;
  const long long base = __shfl_sync(0xffffffffu, off - (long long)excl, 0);  // offsets[s0]
  if (total == 0) return;
  if (base + total > cap) {
    if (lane == 0) atomicOr(&counters[XG_CTR_STATUS], XG_ST_ENTRY_OVERFLOW);
    return;
  }
  const int w = cnt ? (int)(r.z - r.x + 1) : 1;
  for (uint32_t e0 = 0; e0 < total; e0 += 32) {
    const uint32_t e = e0 + lane;
    // owner: the last lane whose exclusive prefix is <= e (binary search via shuffles)
    int lo = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int cand = lo + step;
      const uint32_t ex = __shfl_sync(0xffffffffu, excl, cand & 31);
      if (cand < 32 && ex <= e) lo = cand;
    }
    const uint32_t j = e - __shfl_sync(0xffffffffu, excl, lo);
    const int ow = __shfl_sync(0xffffffffu, w, lo);
    const int ox = __shfl_sync(0xffffffffu, (int)r.x, lo);
    const int oy = __shfl_sync(0xffffffffu, (int)r.y, lo);
    const uint32_t og = __shfl_sync(0xffffffffu, g, lo);
    if (e < total) {
      const int ty = oy + (int)(j / (uint32_t)ow), tx = ox + (int)(j % (uint32_t)ow);
      keys[base + e] = (uint32_t)(ty * ntx + tx);
      vals[base + e] = og;
    }
  }
}

// Tile ranges from the tile-sorted keys: a boundary pass writes the start /
// end of every non-empty tile, then empty tiles get start = end = the start
// of the next non-empty tile (np.searchsorted semantics, frontend.py:171-173).
__global__ void k_tile_bounds(const uint32_t* __restrict__ keys, const uint32_t* counters, long long cap,
                              long long* __restrict__ ranges) {
  long long e = counters[XG_CTR_ENTRIES];
  if (e > cap) e = 0;  // overflow: the list is partial (k_duplicate skips warps past cap); re-binned
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < e;
       k += (long long)gridDim.x * blockDim.x) {
    const uint32_t t = keys[k];
    if (k == 0 || keys[k - 1] != t) ranges[2 * t] = k;
    if (k == e - 1 || keys[k + 1] != t) ranges[2 * t + 1] = k + 1;
  }
}

// Fill empty tiles (pre-set to -1) with the start of the next non-empty
// tile: a suffix-min over tiles, in chunks of 1024 from the back.
__global__ void __launch_bounds__(1024) k_tile_fill(const uint32_t* counters, long long cap, int n_tiles,
                                                    long long* __restrict__ ranges) {
  __shared__ long long s_val[1024];
  __shared__ long long s_next;
  long long e = counters[XG_CTR_ENTRIES];
  if (e > cap) e = 0;  // overflow: every tile empty until the re-bin
  if (threadIdx.x == 0) s_next = e;
  for (int hi = n_tiles; hi > 0; hi -= 1024) {
    const int t = hi - 1024 + (int)threadIdx.x;
    const long long st = t >= 0 ? ranges[2 * t] : -1;
    s_val[threadIdx.x] = st >= 0 ? st : LLONG_MAX;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive suffix min (Hillis-Steele)
      const long long other = threadIdx.x + o < 1024 ? s_val[threadIdx.x + o] : LLONG_MAX;
      __syncthreads();
      if (other < s_val[threadIdx.x]) s_val[threadIdx.x] = other;
      __syncthreads();
    }
    if (t >= 0 && st < 0) {
      long long cand = threadIdx.x + 1 < 1024 ? s_val[threadIdx.x + 1] : LLONG_MAX;
      if (cand == LLONG_MAX) cand = s_next;
      ranges[2 * t] = cand;
      ranges[2 * t + 1] = cand;
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_val[0] != LLONG_MAX) s_next = s_val[0];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Fused duplicate + stable tile sort ("multisplit" counting sort).  The
// depth-sorted Gaussians are cut into chunks of 256 x rounds (one CTA each);
// every Gaussian contributes one entry per tile of its rect.  Pass 1 counts
// entries per (tile, chunk); an exclusive scan over the tile-major table
// gives each (tile, chunk) its output base - and the tile ranges for free.
// Pass 2 re-enumerates the chunk's entries in (depth, rect) order and ranks
// them stably per tile (per-warp counters + __match_any_sync within each
// 32-entry window), writing entry_splat[] directly in (tile, depth, index)
// order.  Replaces writing E (key, value) pairs and two radix passes over
// them with one read of the rects and one write of the values.
// ---------------------------------------------------------------------------
#ifndef XG_BIN_THREADS
#define XG_BIN_THREADS 256
#endif
constexpr int kBinThreads = XG_BIN_THREADS;
constexpr int kBinWarps = kBinThreads / 32;
#ifndef XG_BIN_MAX_ROUNDS
#define XG_BIN_MAX_ROUNDS 16
#endif
constexpr int kBinMaxRounds = XG_BIN_MAX_ROUNDS;              // 32-Gaussian rounds per warp (max)
static_assert(kBinThreads * kBinMaxRounds < 65536, "k_bin_emit keeps per-tile local offsets in 16 bits");

// Rounds per warp (chunk = 256 x rounds Gaussians per CTA).  Every CTA pays
// O(T) fixed work (zeroing and scanning its 8 x T per-warp counters, reading
// T offsets), so the chunk grows with the tile count: ~3 CTAs per SM for
// T <= 1024 (small training clouds still fill the GPU), ~2 waves of one
// CTA per SM (128 KB of counters) at T = 4096.
// (T <= 1024: since single-view training frames take the entry-balanced
// kernels, the chunked ones serve concurrent sweeps, where fewer, longer
// CTAs win - measured on C3: 444 CTAs / <= 4 rounds 2,951 fps, 222 / 8
// 2,978, 160 / 12 2,970, 148 / 16 2,948)
#ifndef XG_BIN_CTAS_SMALL_T
#define XG_BIN_CTAS_SMALL_T 222
#endif
#ifndef XG_BIN_SMALL_T_MAX_ROUNDS
#define XG_BIN_SMALL_T_MAX_ROUNDS 8
#endif
#ifndef XG_BIN_CTAS_LARGE_T
#define XG_BIN_CTAS_LARGE_T 296
#endif
// lat: a single-view (training) frame's chunking - round 1's 444 CTAs of
// up to 4 rounds for T <= 1024 (sweeps take the fewer, longer CTAs above)
inline int bin_rounds(int64_t n, int n_tiles, bool lat = false) {
  const int64_t ctas = n_tiles > 1024 ? XG_BIN_CTAS_LARGE_T : (lat ? 444 : XG_BIN_CTAS_SMALL_T);
  const int64_t r = (n + (int64_t)kBinThreads * ctas - 1) / ((int64_t)kBinThreads * ctas);
  const int cap = n_tiles > 1024 ? kBinMaxRounds : (lat ? 4 : XG_BIN_SMALL_T_MAX_ROUNDS);
  return r < 1 ? 1 : (r > cap ? cap : (int)r);
}
inline int64_t bin_chunk(int64_t n, int n_tiles, bool lat = false) {
  return (int64_t)kBinThreads * bin_rounds(n, n_tiles, lat);
}
constexpr int kBinMaxTiles = 4096;                             // smem: 8 warps x 4096 x 4 B
// k_bin_emit phase 3: (=1, default) a lane per Gaussian with the round's
// peers ranked by column / row lane masks, or (=0) 32-entry windows over the
// round's concatenated entries ranked with __match_any_sync.  The masks take
// 14 % fewer instructions but each lane's walk over its rect is a serial
// shared-memory chain: measured +2.3 % C4 and +0.5 % C3 (sweeps: many views
// hide the chains), -6 % per C2 iteration - which is why single-view
// training frames take the entry-balanced k_bin_emit_bal instead
#ifndef XG_BIN_EMIT_MASKS
#define XG_BIN_EMIT_MASKS 1
#endif

// A warp's 32 depth-sorted Gaussians of one round, software-pipelined: the
// order[] index two rounds ahead and the (count, rect) gather one round ahead
// are issued before the current round is processed.
struct BinLane {
  uint32_t g, cnt;
  uint2 r;  // the ushort4 rect as two words: x0 | y0 << 16, x1 | y1 << 16
  __device__ __forceinline__ int x0() const { return (int)(r.x & 0xffffu); }
  __device__ __forceinline__ int y0() const { return (int)(r.x >> 16); }
  __device__ __forceinline__ int x1() const { return (int)(r.y & 0xffffu); }
  __device__ __forceinline__ int y1() const { return (int)(r.y >> 16); }
};

struct BinPipe {
  const uint32_t* order;
  const uint32_t* n_tiles;
  const ushort4* rect;
  long long n, wlo;
  int lane;
  uint32_t g_next;  // order[] of round rd + 1

  __device__ __forceinline__ uint32_t index(int rd) const {
    const long long s = wlo + rd * 32 + lane;
    return s < n ? order[s] : 0xffffffffu;
  }
  __device__ __forceinline__ BinLane gather(uint32_t g) const {
    BinLane b{g, 0u, make_uint2(0u, 0u)};
    if (g != 0xffffffffu) {
      b.cnt = n_tiles[g];
      b.r = reinterpret_cast<const uint2*>(rect)[g];  // (unused when cnt == 0)
    }
    return b;
  }
  __device__ __forceinline__ BinLane first() {
    const uint32_t g0 = index(0);
    g_next = index(1);
    return gather(g0);
  }
  // the lanes of round rd + 1, given rd + 1 < rounds (prefetches rd + 2)
  __device__ __forceinline__ BinLane next(int rd) {
    const BinLane b = gather(g_next);
    g_next = index(rd + 2);
    return b;
  }
};

// Per-warp entry counts per tile, 16-bit, two tiles per word
// ([C][kBinWarps][ceil(T/2)], the warp's Gaussians exactly as k_bin_emit
// walks them), kept for k_bin_emit, and the per-CTA totals hist[T][C] for
// the scan.
__global__ void __launch_bounds__(kBinThreads)
    k_bin_count(const uint32_t* __restrict__ order, const uint32_t* __restrict__ n_tiles,
                const ushort4* __restrict__ rect, long long n, int ntx, int T, int rounds,
                uint32_t* __restrict__ hist, uint32_t* __restrict__ wc_out) {
  extern __shared__ uint32_t wcnt[];  // [kBinWarps][TW]
  const int TW = (T + 1) >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kBinWarps * TW; i += kBinThreads) wcnt[i] = 0;
  __syncthreads();
  uint32_t* mine = wcnt + warp * TW;
  const long long wlo = (long long)blockIdx.x * kBinThreads * rounds + (long long)warp * 32 * rounds;
  BinPipe pipe{order, n_tiles, rect, n, wlo, lane, 0u};
  BinLane cur = pipe.first();
  for (int rd = 0; rd < rounds; ++rd) {
    BinLane nxt{};
    if (rd + 1 < rounds) nxt = pipe.next(rd);
    if (cur.cnt) {
      const int x0 = cur.x0(), y0 = cur.y0(), x1 = cur.x1(), y1 = cur.y1();
      for (int ty = y0; ty <= y1; ++ty)
        for (int tx = x0; tx <= x1; ++tx) {
          const int t = ty * ntx + tx;
          atomicAdd(&mine[t >> 1], 1u << ((t & 1) << 4));
        }
    }
    cur = nxt;
  }
  __syncthreads();
  const int C = gridDim.x;
  uint32_t* out = wc_out + (long long)blockIdx.x * kBinWarps * TW;
  for (int k = threadIdx.x; k < TW; k += kBinThreads) {
    uint32_t s0 = 0, s1 = 0;
#pragma unroll
    for (int w = 0; w < kBinWarps; ++w) {
      const uint32_t c = wcnt[w * TW + k];
      out[w * TW + k] = c;
      s0 += c & 0xffffu;
      s1 += c >> 16;
    }
    hist[(long long)(2 * k) * C + blockIdx.x] = s0;
    if (2 * k + 1 < T) hist[(long long)(2 * k + 1) * C + blockIdx.x] = s1;
  }
}

// (tile ranges from the scanned (tile, chunk) table; thread 0 also flags an
// entry-buffer overflow, which only needs the scan's total)
__global__ void k_bin_ranges(const uint32_t* __restrict__ offs, int C, int T, uint32_t* counters, long long cap,
                             long long* __restrict__ ranges) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0 && (long long)counters[XG_CTR_ENTRIES] > cap) atomicOr(&counters[XG_CTR_STATUS], XG_ST_ENTRY_OVERFLOW);
  if (t >= T) return;
  ranges[2 * t] = offs[(long long)t * C];
  ranges[2 * t + 1] = t + 1 < T ? (long long)offs[(long long)(t + 1) * C] : (long long)counters[XG_CTR_ENTRIES];
}

// T <= 1024: k_bin_ranges and the compositing schedule (k_tile_order's
// heaviest-first order, same 64 log-spaced buckets) in one CTA - one launch
// fewer per view
__global__ void __launch_bounds__(1024) k_bin_ranges_order(const uint32_t* __restrict__ offs, int C, int T,
                                                           uint32_t* counters, long long cap,
                                                           long long* __restrict__ ranges, int* __restrict__ order) {
  constexpr int NB = 64;
  __shared__ int hist[NB];
  __shared__ int off[NB];
  const int t = threadIdx.x;
  if (t < NB) hist[t] = 0;
  const long long E = (long long)counters[XG_CTR_ENTRIES];
  if (t == 0 && E > cap) atomicOr(&counters[XG_CTR_STATUS], XG_ST_ENTRY_OVERFLOW);
  long long s0 = 0, s1 = 0;
  if (t < T) {
    s0 = offs[(long long)t * C];
    s1 = t + 1 < T ? (long long)offs[(long long)(t + 1) * C] : E;
    ranges[2 * t] = s0;
    ranges[2 * t + 1] = s1;
  }
  const long long len = s1 - s0;
  const int b = len > 0 ? (int)(4.f * __log2f((float)len + 1.f)) : 0;
  const int key = NB - 1 - min(b, NB - 1);
  __syncthreads();
  if (t < T) atomicAdd(&hist[key], 1);
  __syncthreads();
  if (t == 0) {
    int run = 0;
    for (int k = 0; k < NB; ++k) {
      off[k] = run;
      run += hist[k];
    }
  }
  __syncthreads();
  if (t < T) order[atomicAdd(&off[key], 1)] = t;
}

__global__ void __launch_bounds__(kBinThreads)
    k_bin_emit(const uint32_t* __restrict__ order, const uint32_t* __restrict__ n_tiles,
               const ushort4* __restrict__ rect, long long n, int ntx, int T, int rounds,
               const uint32_t* __restrict__ offs, const uint32_t* __restrict__ wc_in, long long cap,
               uint32_t* __restrict__ entry_splat) {
  // shared: base[T] (the CTA's global start per tile, 32-bit) and per-warp
  // 16-bit counters / local offsets packed two tiles per word
  // ([kBinWarps][ceil(T/2)]): 20 T bytes, so two CTAs fit an SM at T = 4096.
  // Local offsets are bounded by the chunk (<= 256 x 16 Gaussians, one entry
  // per tile each) and stay below 2^16.
  extern __shared__ uint32_t smem_bin[];
  const int TW = (T + 1) >> 1;
  uint32_t* tbase = smem_bin;
  uint32_t* wcnt = smem_bin + T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = gridDim.x;
  // phase 1: the per-warp counts k_bin_count kept
  const uint32_t* wc = wc_in + (long long)blockIdx.x * kBinWarps * TW;
  for (int i = threadIdx.x; i < kBinWarps * TW; i += kBinThreads) wcnt[i] = wc[i];
  __syncthreads();
  uint32_t* mine = wcnt + warp * TW;
  uint16_t* mine16 = reinterpret_cast<uint16_t*>(mine);  // tile t = half t & 1 of word t >> 1 (little endian)
  const long long wlo = (long long)blockIdx.x * kBinThreads * rounds + (long long)warp * 32 * rounds;
  // phase 2: the CTA's global base per tile, per-warp local offsets (a thread
  // owns one word = two tiles)
  for (int k = threadIdx.x; k < TW; k += kBinThreads) {
    const int t0 = 2 * k, t1 = 2 * k + 1;
    tbase[t0] = offs[(long long)t0 * C + blockIdx.x];
    if (t1 < T) tbase[t1] = offs[(long long)t1 * C + blockIdx.x];
    uint32_t l0 = 0, l1 = 0;
    for (int w = 0; w < kBinWarps; ++w) {
      const uint32_t c = wcnt[w * TW + k];
      wcnt[w * TW + k] = l0 | (l1 << 16);
      l0 += c & 0xffffu;
      l1 += c >> 16;
    }
  }
  __syncthreads();
#if XG_BIN_EMIT_MASKS
  // phase 3: each lane walks its own Gaussian's rect.  A tile's peers in the
  // round (the lanes whose rects contain it, lane order = depth order) are
  // the AND of two per-warp bit masks, column and row, built with one shared
  // OR per rect column and row; the entry's rank among them is a popcount.
  // A tile only this lane covers updates its local offset at once; shared
  // tiles are advanced by their highest peer after the round's writes.
  const int nty = T / ntx;
  uint32_t* cmask = smem_bin + T + kBinWarps * TW + warp * (ntx + nty);
  uint32_t* rmask = cmask + ntx;
  const unsigned lt = lanemask_lt(), bit = 1u << lane;
  const uint32_t cap32 = cap < 0xffffffffll ? (uint32_t)cap : 0xffffffffu;
  BinPipe pipe{order, n_tiles, rect, n, wlo, lane, 0u};
  BinLane cur = pipe.first();
  for (int rd = 0; rd < rounds; ++rd) {
    BinLane nxt{};
    if (rd + 1 < rounds) nxt = pipe.next(rd);
    const uint32_t g = cur.g, cnt = cur.cnt;
    const int x0 = cur.x0(), y0 = cur.y0(), x1 = cur.x1(), y1 = cur.y1();
    for (int k = lane; k < ntx + nty; k += 32) cmask[k] = 0u;
    __syncwarp();
    if (cnt) {
      for (int x = x0; x <= x1; ++x) atomicOr(&cmask[x], bit);
      for (int y = y0; y <= y1; ++y) atomicOr(&rmask[y], bit);
    }
    __syncwarp();
    bool shared_tiles = false;
    if (cnt) {
      for (int y = y0; y <= y1; ++y) {
        const uint32_t rm = rmask[y];
        for (int x = x0; x <= x1; ++x) {
          const uint32_t peers = rm & cmask[x];
          const int t = y * ntx + x;
          const uint32_t loc = mine16[t];
          const uint32_t pos = tbase[t] + loc + (uint32_t)__popc(peers & lt);
          if (pos < cap32) entry_splat[pos] = g;
          if (peers == bit)
            mine16[t] = (uint16_t)(loc + 1u);
          else
            shared_tiles = true;
        }
      }
    }
    if (__any_sync(0xffffffffu, shared_tiles)) {
      __syncwarp();
      if (shared_tiles) {
        for (int y = y0; y <= y1; ++y) {
          const uint32_t rm = rmask[y];
          for (int x = x0; x <= x1; ++x) {
            const uint32_t peers = rm & cmask[x];
            if (peers != bit && (peers >> lane) == 1u) {
              const int t = y * ntx + x;
              mine16[t] = (uint16_t)(mine16[t] + (uint32_t)__popc(peers));
            }
          }
        }
      }
    }
    __syncwarp();
    cur = nxt;
  }
}
#else
  // phase 3: enumerate entries in (depth, rect row-major) order, rank per tile
  __shared__ uint32_t s_nz[kBinWarps][32];  // lanes with entries, in lane order
  const unsigned lt = lanemask_lt();
  BinPipe pipe{order, n_tiles, rect, n, wlo, lane, 0u};
  BinLane cur = pipe.first();
  for (int rd = 0; rd < rounds; ++rd) {
    BinLane nxt{};
    if (rd + 1 < rounds) nxt = pipe.next(rd);
    const uint32_t g = cur.g, cnt = cur.cnt;
    const ushort4 r = make_ushort4((uint16_t)cur.x0(), (uint16_t)cur.y0(), (uint16_t)cur.x1(), (uint16_t)cur.y1());
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - cnt;
    const int wdt = cnt ? (int)(r.z - r.x + 1) : 1;
    // j / wdt as a multiply-high: exact for j, wdt < 2^16 with m = ceil(2^32 / wdt)
    // (wdt = 1, where m would be 2^32, is marked by m = 0)
    const uint32_t mdiv =
        wdt > 1 ? (uint32_t)((0x100000000ull + (unsigned long long)wdt - 1ull) / (unsigned long long)wdt) : 0u;
    // owner of entry e = the last lane with entries whose exclusive prefix is
    // <= e: per 32-entry window, the lanes' start positions as one bit mask
    // (redux.sync.or) and the count of starts up to e index the compacted
    // list of lanes with entries (no dependent shuffle chain)
    const unsigned nzm = __ballot_sync(0xffffffffu, cnt > 0);
    if (cnt > 0) s_nz[warp][__popc(nzm & lt)] = (uint32_t)lane;
    __syncwarp();
    uint32_t before = 0;  // starts before the window
    for (uint32_t e0 = 0; e0 < total; e0 += 32) {
      const uint32_t e = e0 + lane;
      const uint32_t bit = (cnt > 0 && excl >= e0 && excl - e0 < 32u) ? 1u << (excl - e0) : 0u;
      const uint32_t starts = __reduce_or_sync(0xffffffffu, bit);
      const uint32_t R = before + __popc(starts & (0xffffffffu >> (31 - lane)));  // starts <= e (>= 1)
      before += __popc(starts);
      const int lo = (int)s_nz[warp][R - 1u];
      const uint32_t j = e - __shfl_sync(0xffffffffu, excl, lo);
      const int ow = __shfl_sync(0xffffffffu, wdt, lo);
      const uint32_t om = __shfl_sync(0xffffffffu, mdiv, lo);
      const int ox = __shfl_sync(0xffffffffu, (int)r.x, lo);
      const int oy = __shfl_sync(0xffffffffu, (int)r.y, lo);
      const uint32_t og = __shfl_sync(0xffffffffu, g, lo);
      const bool valid = e < total;
      const uint32_t jq = om ? __umulhi(j, om) : j;
      const int t = valid ? (oy + (int)jq) * ntx + ox + (int)(j - jq * (uint32_t)ow) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, t);
      const uint32_t loc = valid ? (uint32_t)mine16[t] : 0u;
      if (valid) {
        const long long pos = (long long)tbase[t] + loc + __popc(peers & lt);
        if (pos < cap) entry_splat[pos] = og;
      }
      __syncwarp();
      if (valid && (peers >> lane) == 1u) mine16[t] = (uint16_t)(loc + __popc(peers));  // highest peer lane
      __syncwarp();
    }
    __syncwarp();  // (s_nz is rewritten by the next round)
    cur = nxt;
  }
}
#endif

// ---------------------------------------------------------------------------
// Entry-balanced multisplit (T <= XG_BIN_BAL_TILES).  The Gaussian-chunked
// kernels above give every warp 32 x rounds depth-sorted Gaussians, so one
// warp of large splats walks thousands of entries while its neighbours walk
// hundreds: on a trained C2 cloud (tiles touched p50 16, p99 132, max 1,024)
// the slowest warp holds 4.3x the median's entries and the emit ran with its
// SMs active 56 % of the time.  Here the scan of tiles-touched in depth order (offN, the
// entries' global offsets) cuts the E entries into C x 8 equal warp slices:
// warp w of CTA c walks entries [c EC + w EC / 8, ...) in the same (depth,
// rect row-major) order - so per-(CTA, warp, tile) counts still rank every
// entry stably - whatever splats they belong to.  The owner of the slice's
// first entry comes from a 32-ary search of offN (k_bin_count_bal, stored
// per warp for k_bin_emit_bal).
// ---------------------------------------------------------------------------
#ifndef XG_BIN_BAL_TILES
#define XG_BIN_BAL_TILES 1024
#endif
#ifndef XG_BIN_BAL_CTAS
#define XG_BIN_BAL_CTAS 444
#endif
#ifndef XG_BIN_COUNT_MATCH
#define XG_BIN_COUNT_MATCH 0
#endif

// entries per CTA: a multiple of 8 x 32, <= 65280 while E <= C x 65280
__device__ __forceinline__ uint32_t bal_chunk(uint32_t E, int C) {
  const uint32_t per = (uint32_t)(((unsigned long long)E + (unsigned long long)C - 1ull) / (unsigned long long)C);
  return (per + 255u) & ~255u;
}

// first s in [0, n) with offN[s] > x (n if none): 32-ary warp search
__device__ __forceinline__ long long upper_bound_warp(const uint32_t* __restrict__ offN, long long n, uint32_t x,
                                                      int lane) {
  long long a = 0, b = n;  // answer in [a, b]
  while (b - a > 32) {
    const long long step = (b - a + 31) / 32;
    const long long p = a + (long long)lane * step;
    const bool gt = p >= b || offN[p] > x;
    const unsigned m = __ballot_sync(0xffffffffu, gt);
    const int j = m ? __ffs(m) - 1 : 32;
    if (j == 0) return a;  // (offN[a] > x)
    const long long pj1 = a + (long long)(j - 1) * step;
    b = j < 32 ? min(b, a + (long long)j * step) : b;
    a = pj1 + 1;
  }
  const long long p = a + lane;
  const unsigned m = __ballot_sync(0xffffffffu, p < b && offN[p] > x);
  return m ? a + (__ffs(m) - 1) : b;
}

// Walks entries [lo, hi) of the depth-ordered entry sequence with the warp,
// 32 at a time, starting at depth-sorted Gaussian s_first (the owner of
// entry lo): f(valid, tile, gaussian) per lane and window (every lane calls
// f, so f may use warp collectives).
template <class F>
__device__ __forceinline__ void walk_entries(const uint32_t* __restrict__ order, const uint32_t* __restrict__ n_tiles,
                                             const ushort4* __restrict__ rect, const uint32_t* __restrict__ offN,
                                             long long n, int ntx, uint32_t lo, uint32_t hi, long long s_first,
                                             uint32_t* s_nz, F&& f) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  // software pipeline: the next round's (order, offset) one round ahead
  long long s0 = s_first;
  uint32_t g_n = 0xffffffffu, off_n = 0;
  {
    const long long s = s0 + lane;
    if (s < n) {
      g_n = order[s];
      off_n = offN[s];
    }
  }
  while (lo < hi && s0 < n) {
    const uint32_t g = g_n, off = off_n;
    uint32_t cnt = 0;
    uint2 rr = make_uint2(0u, 0u);
    if (g != 0xffffffffu) {
      cnt = n_tiles[g];
      if (cnt) rr = reinterpret_cast<const uint2*>(rect)[g];
    }
    {
      const long long s = s0 + 32 + lane;
      g_n = 0xffffffffu;
      if (s < n) {
        g_n = order[s];
        off_n = offN[s];
      }
    }
    const uint32_t base = __shfl_sync(0xffffffffu, off, 0);
    if (base >= hi) break;
    const uint32_t excl = off - base;
    // the round's entry count (lanes past n carry stale offsets: only lanes with entries count)
    const uint32_t incl_last = __reduce_max_sync(0xffffffffu, cnt > 0 ? excl + cnt : 0u);
    const uint32_t rs = lo - base;  // (base <= lo: base is the owner's or the previous round's end)
    const uint32_t re = min(hi - base, incl_last);
    const int x0 = (int)(rr.x & 0xffffu), y0 = (int)(rr.x >> 16), x1 = (int)(rr.y & 0xffffu);
    const int wdt = cnt ? x1 - x0 + 1 : 1;
    const uint32_t mdiv =
        wdt > 1 ? (uint32_t)((0x100000000ull + (unsigned long long)wdt - 1ull) / (unsigned long long)wdt) : 0u;
    const unsigned nzm = __ballot_sync(0xffffffffu, cnt > 0);
    if (cnt > 0) s_nz[__popc(nzm & lt)] = (uint32_t)lane;
    __syncwarp();
    uint32_t before = __popc(__ballot_sync(0xffffffffu, cnt > 0 && excl < rs));  // starts before the first window
    for (uint32_t e0 = rs; e0 < re; e0 += 32) {
      const uint32_t e = e0 + lane;
      const uint32_t bit = (cnt > 0 && excl >= e0 && excl - e0 < 32u) ? 1u << (excl - e0) : 0u;
      const uint32_t starts = __reduce_or_sync(0xffffffffu, bit);
      const uint32_t R = before + __popc(starts & (0xffffffffu >> (31 - lane)));  // starts <= e (>= 1)
      before += __popc(starts);
      const int ol = (int)s_nz[R - 1u];
      const uint32_t j = e - __shfl_sync(0xffffffffu, excl, ol);
      const int ow = __shfl_sync(0xffffffffu, wdt, ol);
      const uint32_t om = __shfl_sync(0xffffffffu, mdiv, ol);
      const int ox = __shfl_sync(0xffffffffu, x0, ol);
      const int oy = __shfl_sync(0xffffffffu, y0, ol);
      const uint32_t og = __shfl_sync(0xffffffffu, g, ol);
      const bool valid = e < re;
      const uint32_t jq = om ? __umulhi(j, om) : j;
      const int t = valid ? (oy + (int)jq) * ntx + ox + (int)(j - jq * (uint32_t)ow) : -1;
      f(valid, t, og);
    }
    __syncwarp();  // (s_nz is rewritten by the next round)
    lo = base + incl_last;
    s0 += 32;
  }
}

__global__ void __launch_bounds__(kBinThreads)
    k_bin_count_bal(const uint32_t* __restrict__ order, const uint32_t* __restrict__ n_tiles,
                    const ushort4* __restrict__ rect, const uint32_t* __restrict__ offN, long long n, int ntx, int T,
                    const uint32_t* __restrict__ n_entries, uint32_t* __restrict__ hist,
                    uint32_t* __restrict__ wc_out, uint32_t* __restrict__ wstart) {
  extern __shared__ uint32_t wcnt[];  // [kBinWarps][TW]
  __shared__ uint32_t s_nz[kBinWarps][32];
  const int TW = (T + 1) >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kBinWarps * TW; i += kBinThreads) wcnt[i] = 0;
  const int C = gridDim.x;
  const uint32_t E = *n_entries, EC = bal_chunk(E, C), EW = EC / kBinWarps;
  const unsigned long long lo64 = (unsigned long long)blockIdx.x * EC + (unsigned long long)warp * EW;
  const uint32_t lo = (uint32_t)min(lo64, (unsigned long long)E), hi = (uint32_t)min(lo64 + EW, (unsigned long long)E);
  long long s_first = n;
  if (lo < hi) s_first = upper_bound_warp(offN, n, lo, lane) - 1;
  if (lane == 0) wstart[blockIdx.x * kBinWarps + warp] = (uint32_t)s_first;
  __syncthreads();
  uint32_t* mine = wcnt + warp * TW;
  walk_entries(order, n_tiles, rect, offN, n, ntx, lo, hi, s_first, s_nz[warp], [&](bool valid, int t, uint32_t) {
#if XG_BIN_COUNT_MATCH
    const unsigned peers = __match_any_sync(0xffffffffu, t);
    if (valid && (peers >> lane) == 1u) atomicAdd(&mine[t >> 1], (uint32_t)__popc(peers) << ((t & 1) << 4));
#else
    // (a window's entries mostly hit distinct tiles - one splat's rect row -
    // so plain shared atomics beat aggregating peers first)
    if (valid) atomicAdd(&mine[t >> 1], 1u << ((t & 1) << 4));
#endif
  });
  __syncthreads();
  uint32_t* out = wc_out + (long long)blockIdx.x * kBinWarps * TW;
  for (int k = threadIdx.x; k < TW; k += kBinThreads) {
    uint32_t s0 = 0, s1 = 0;
#pragma unroll
    for (int w = 0; w < kBinWarps; ++w) {
      const uint32_t c = wcnt[w * TW + k];
      out[w * TW + k] = c;
      s0 += c & 0xffffu;
      s1 += c >> 16;
    }
    hist[(long long)(2 * k) * C + blockIdx.x] = s0;
    if (2 * k + 1 < T) hist[(long long)(2 * k + 1) * C + blockIdx.x] = s1;
  }
}

__global__ void __launch_bounds__(kBinThreads)
    k_bin_emit_bal(const uint32_t* __restrict__ order, const uint32_t* __restrict__ n_tiles,
                   const ushort4* __restrict__ rect, const uint32_t* __restrict__ offN, long long n, int ntx, int T,
                   const uint32_t* __restrict__ n_entries, const uint32_t* __restrict__ offs,
                   const uint32_t* __restrict__ wc_in, const uint32_t* __restrict__ wstart, long long cap,
                   uint32_t* __restrict__ entry_splat) {
  extern __shared__ uint32_t smem_bin[];
  __shared__ uint32_t s_nz[kBinWarps][32];
  const int TW = (T + 1) >> 1;
  uint32_t* tbase = smem_bin;
  uint32_t* wcnt = smem_bin + T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = gridDim.x;
  const uint32_t* wc = wc_in + (long long)blockIdx.x * kBinWarps * TW;
  for (int i = threadIdx.x; i < kBinWarps * TW; i += kBinThreads) wcnt[i] = wc[i];
  __syncthreads();
  for (int k = threadIdx.x; k < TW; k += kBinThreads) {
    const int t0 = 2 * k, t1 = 2 * k + 1;
    tbase[t0] = offs[(long long)t0 * C + blockIdx.x];
    if (t1 < T) tbase[t1] = offs[(long long)t1 * C + blockIdx.x];
    uint32_t l0 = 0, l1 = 0;
    for (int w = 0; w < kBinWarps; ++w) {
      const uint32_t c = wcnt[w * TW + k];
      wcnt[w * TW + k] = l0 | (l1 << 16);
      l0 += c & 0xffffu;
      l1 += c >> 16;
    }
  }
  __syncthreads();
  const uint32_t E = *n_entries, EC = bal_chunk(E, C), EW = EC / kBinWarps;
  const unsigned long long lo64 = (unsigned long long)blockIdx.x * EC + (unsigned long long)warp * EW;
  const uint32_t lo = (uint32_t)min(lo64, (unsigned long long)E), hi = (uint32_t)min(lo64 + EW, (unsigned long long)E);
  uint16_t* mine16 = reinterpret_cast<uint16_t*>(wcnt + warp * TW);
  const unsigned lt = lanemask_lt();
  const long long s_first = lo < hi ? (long long)wstart[blockIdx.x * kBinWarps + warp] : n;
  walk_entries(order, n_tiles, rect, offN, n, ntx, lo, hi, s_first, s_nz[warp], [&](bool valid, int t, uint32_t og) {
    const unsigned peers = __match_any_sync(0xffffffffu, t);
    const uint32_t loc = valid ? (uint32_t)mine16[t] : 0u;
    if (valid) {
      const long long pos = (long long)tbase[t] + loc + __popc(peers & lt);
      if (pos < cap) entry_splat[pos] = og;
    }
    __syncwarp();
    if (valid && (peers >> lane) == 1u) mine16[t] = (uint16_t)(loc + __popc(peers));  // highest peer lane
    __syncwarp();
  });
}

struct BinWs {
  unsigned long long *keyN1, *keyN2;
  uint32_t *valN1, *offN, *keyE0, *keyE1, *valE1;
  uint32_t *hist, *hoff;  // multisplit path: [T][C] counts and their scan
  uint32_t* wcnt;         //   and the per-warp 16-bit counts [C][kBinWarps][ceil(T/2)]
  uint32_t* wstart;       //   balanced path: each warp's first depth-sorted splat [C][kBinWarps]
  void* tail;
  size_t tail_bytes;
};

// fused multisplit up to this many tiles, duplicate + radix sort beyond
#ifndef XG_BIN_MULTISPLIT_TILES
#define XG_BIN_MULTISPLIT_TILES 4096
#endif
static_assert(XG_BIN_MULTISPLIT_TILES <= 4096, "multisplit counters: 8 warps x 4096 x 4 B of shared memory");
bool multisplit(int n_tiles) { return n_tiles <= XG_BIN_MULTISPLIT_TILES; }

int64_t bin_chunks(int64_t n, int n_tiles, bool lat = false) {
  return (n + bin_chunk(n, n_tiles, lat) - 1) / bin_chunk(n, n_tiles, lat);
}

// entry-balanced count / emit (XG_BIN_BALANCED=0 selects the Gaussian-chunked kernels)
// (1: training frames, 2: every frame, 0: never)
int bal_mode() {
  static const int m = getenv("XG_BIN_BALANCED") ? atoi(getenv("XG_BIN_BALANCED")) : 1;
  return m;
}
bool balanced(int n_tiles) { return bal_mode() && n_tiles <= XG_BIN_BAL_TILES; }
// balanced grid: XG_BIN_BAL_CTAS, more if the capacity needs it (entries per
// CTA stay below 2^16: 16-bit local offsets)
int64_t bal_grid(int64_t cap) {
  const int64_t need = (cap + 65279) / 65280;
  return need > XG_BIN_BAL_CTAS ? need : XG_BIN_BAL_CTAS;
}
// CTAs of the multisplit count / emit launches (the (tile, chunk) table
// width) - workspaces are sized for either path
int64_t ms_chunks(int64_t n, int64_t cap, int n_tiles) {
  int64_t a = bin_chunks(n, n_tiles);
  const int64_t al = bin_chunks(n, n_tiles, true);
  if (al > a) a = al;
  if (!balanced(n_tiles)) return a;
  const int64_t b = bal_grid(cap);
  return a > b ? a : b;
}

size_t bin_wcnt_bytes(int64_t n, int64_t cap, int n_tiles) {
  if (!multisplit(n_tiles)) return 0;
  const int64_t C = ms_chunks(n, cap, n_tiles);
  return align_up(sizeof(uint32_t) * (size_t)C * kBinWarps * (size_t)((n_tiles + 1) / 2)) +
         align_up(sizeof(uint32_t) * (size_t)C * kBinWarps);  // (+ the balanced path's per-warp start splats)
}

size_t tail_bytes(int64_t n, int64_t cap, int n_tiles) {
  size_t a = radix_workspace_bytes(multisplit(n_tiles) ? n : (n > cap ? n : cap));
  const size_t o = onesweep_workspace_bytes(n);
  if (o > a) a = o;
  const size_t bsw = bucket_sort_workspace_bytes(n);
  if (bsw > a) a = bsw;
  const int64_t hn = multisplit(n_tiles) ? (int64_t)n_tiles * ms_chunks(n, cap, n_tiles) : 0;
  // (balanced path: the offsets scan and the (tile, chunk) scan side by side, cleared by one memset)
  size_t b = align_up(scan_workspace_bytes(n)) + align_up(scan_workspace_bytes(hn > 0 ? hn : 1));
  return a > b ? a : b;
}

bool carve(void* ws, size_t bytes, int64_t n, int64_t cap, int n_tiles, BinWs& w) {
  char* p = (char*)ws;
  const size_t bn = align_up(sizeof(uint32_t) * (size_t)n);
  const bool ms = multisplit(n_tiles);
  const size_t be = ms ? 0 : align_up(sizeof(uint32_t) * (size_t)(cap > 0 ? cap : 1));
  const size_t bh = ms ? align_up(sizeof(uint32_t) * (size_t)n_tiles * (size_t)ms_chunks(n, cap, n_tiles)) : 0;
  w.keyN1 = (unsigned long long*)p; p += 2 * bn;
  w.keyN2 = (unsigned long long*)p; p += 2 * bn;
  w.valN1 = (uint32_t*)p; p += bn;
  w.offN = (uint32_t*)p; p += bn;
  w.keyE0 = (uint32_t*)p; p += be;
  w.keyE1 = (uint32_t*)p; p += be;
  w.valE1 = (uint32_t*)p; p += be;
  w.hist = (uint32_t*)p; p += bh;
  w.hoff = (uint32_t*)p; p += bh;
  w.wcnt = (uint32_t*)p;
  w.wstart = ms ? (uint32_t*)(p + align_up(sizeof(uint32_t) * (size_t)ms_chunks(n, cap, n_tiles) * kBinWarps *
                                            (size_t)((n_tiles + 1) / 2)))
                : nullptr;
  p += bin_wcnt_bytes(n, cap, n_tiles);
  w.tail = p;
  const size_t used = (size_t)(p - (char*)ws);
  const size_t tb = tail_bytes(n, cap, n_tiles);
  if (used + tb > bytes) return false;
  w.tail_bytes = bytes - used;
  return true;
}

}  // namespace
}  // namespace xg

using namespace xg;

extern "C" {

size_t xg_bin_workspace_bytes(int64_t n, int64_t entry_capacity, int32_t n_tiles_total) {
  const size_t bn = align_up(sizeof(uint32_t) * (size_t)n);
  const bool ms = multisplit(n_tiles_total);
  const size_t be = ms ? 0 : align_up(sizeof(uint32_t) * (size_t)(entry_capacity > 0 ? entry_capacity : 1));
  const size_t bh =
      ms ? align_up(sizeof(uint32_t) * (size_t)n_tiles_total * (size_t)ms_chunks(n, entry_capacity, n_tiles_total)) : 0;
  return 6 * bn + 3 * be + 2 * bh + bin_wcnt_bytes(n, entry_capacity, n_tiles_total) + tail_bytes(n, entry_capacity, n_tiles_total) +
         256;
}

xg_status xg_bin_sort(const xg_camera* cam, xg_splats* sp, void* workspace, size_t workspace_bytes,
                      void* stream) {
  if (!cam || !sp || !workspace || !sp->order || !sp->entry_splat || !sp->tile_ranges ||
      !sp->depth_key || !sp->n_tiles || !sp->rect || !sp->counters || sp->n < 1) {
    set_error_msg("xg_bin_sort: invalid argument");
    return XG_ERR_INVALID;
  }
  BinWs w;
  const int64_t n = sp->n, cap = sp->entry_capacity;
  const int ntx = tiles_x(*cam), nty = tiles_y(*cam);
  const int n_tiles = ntx * nty;
  if (!carve(workspace, workspace_bytes, n, cap, n_tiles, w)) {
    set_error_msg("xg_bin_sort: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  xg_status st;
  // n as a device count for the generic sort: stash it in counters[TOUCH]
  uint32_t* n_dev = sp->counters + XG_CTR_TOUCH;
  // 1. depth sort (depth_key is the sort's read-only input: a re-bin after an
  // entry overflow sorts the same keys again).  Default: the bucket sort
  // (xg_sort.cu); XG_DEPTH_SORT=onesweep selects the 8-pass LSD onesweep.
  static const bool onesweep = getenv("XG_DEPTH_SORT") && strcmp(getenv("XG_DEPTH_SORT"), "onesweep") == 0;
  if (onesweep) {
    k_iota<<<div_up(n, 256), 256, 0, s>>>(sp->order, n, n_dev);
    if ((st = check_launch("k_iota")) != XG_OK) return st;
    if ((st = onesweep_sort_pairs64((const unsigned long long*)sp->depth_key, sp->order, w.keyN1, w.keyN2, w.valN1,
                                    sp->order, sp->order, n, n_dev, w.tail, w.tail_bytes, s)) != XG_OK)
      return st;
  } else if ((st = bucket_sort_depth((const unsigned long long*)sp->depth_key, sp->n_tiles, n, w.keyN1, w.keyN2,
                                     w.valN1, w.offN, sp->order, n_dev, w.tail, w.tail_bytes, s)) != XG_OK) {
    return st;
  }
  // (development aid, tools/probe_bin_graph.py: XG_BIN_STOP=1 stops after
  // the depth sort, 2 after the count / scan / ranges - the stage costs
  // inside a concurrent sweep; results are then incomplete)
  static const int bin_stop = getenv("XG_BIN_STOP") ? atoi(getenv("XG_BIN_STOP")) : 0;
  if (bin_stop == 1) return XG_OK;
  if (multisplit(n_tiles)) {
    // 2-4. fused duplicate + stable tile sort + ranges
    // entry-balanced count / emit for training frames (those with replay
    // checkpoints): one view at a time, so the slowest warp is the launch;
    // sweeps keep the Gaussian-chunked kernels (fewer instructions per entry,
    // their imbalance hidden by the views binned concurrently - measured:
    // balanced C3 -5 %, C2 +1.6 %)
    // (XG_BIN_TRAIN_CHUNKED=1, measurement: training frames on the
    // Gaussian-chunked kernels with the latency chunking)
    static const bool train_chunked = getenv("XG_BIN_TRAIN_CHUNKED") && atoi(getenv("XG_BIN_TRAIN_CHUNKED")) > 0;
    const bool lat = sp->replay_ckpt != nullptr;
    const bool bal = balanced(n_tiles) && (lat || bal_mode() == 2) && !(train_chunked && lat);
    const int rounds = bin_rounds(n, n_tiles, lat);
    const int C = (int)(bal ? bal_grid(cap) : bin_chunks(n, n_tiles, lat));
    void* scan2_ws = nullptr;
    size_t scan2_bytes = 0;
    const size_t sm_count = sizeof(uint32_t) * (size_t)kBinWarps * ((n_tiles + 1) / 2);
    const size_t sm_emit = sizeof(uint32_t) * ((size_t)n_tiles + (size_t)kBinWarps * ((n_tiles + 1) / 2) +
                                               (XG_BIN_EMIT_MASKS ? (size_t)kBinWarps * (ntx + nty) : 0));
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(k_bin_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(uint32_t) * (kBinMaxTiles + kBinWarps * (kBinMaxTiles / 2) +
                                                     (XG_BIN_EMIT_MASKS ? kBinWarps * (kBinMaxTiles + 1) : 0))));
      cudaFuncSetAttribute(k_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(uint32_t) * kBinWarps * (kBinMaxTiles / 2)));
      attr_set = true;
    }
    if (bal) {
      // entry offsets of the depth-sorted splats (and E) cut the entries into equal warp slices
      // both scans' look-back states zeroed by one memset (the depth sort used this space)
      const size_t need1 = align_up(scan_workspace_bytes(n));
      scan2_ws = (char*)w.tail + need1;
      scan2_bytes = w.tail_bytes - need1;
      cudaMemsetAsync(w.tail, 0, need1 + scan_workspace_bytes((long long)n_tiles * C), s);
      scan_u32_precleared_next();
      if ((st = scan_u32(sp->n_tiles, sp->order, w.offN, n, nullptr, n, sp->counters + XG_CTR_ENTRIES, w.tail,
                         need1, s)) != XG_OK)
        return st;
      static bool attr_bal = false;
      if (!attr_bal) {
        cudaFuncSetAttribute(k_bin_emit_bal, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(uint32_t) * (kBinMaxTiles + kBinWarps * (kBinMaxTiles / 2))));
        cudaFuncSetAttribute(k_bin_count_bal, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(uint32_t) * kBinWarps * (kBinMaxTiles / 2)));
        attr_bal = true;
      }
      k_bin_count_bal<<<C, kBinThreads, sm_count, s>>>(sp->order, sp->n_tiles, (const ushort4*)sp->rect, w.offN, n,
                                                       ntx, n_tiles, sp->counters + XG_CTR_ENTRIES, w.hist, w.wcnt,
                                                       w.wstart);
      if ((st = check_launch("k_bin_count_bal")) != XG_OK) return st;
    } else {
      k_bin_count<<<C, kBinThreads, sm_count, s>>>(sp->order, sp->n_tiles, (const ushort4*)sp->rect, n, ntx, n_tiles,
                                                   rounds, w.hist, w.wcnt);
      if ((st = check_launch("k_bin_count")) != XG_OK) return st;
    }
    const long long hn = (long long)n_tiles * C;
    if (bal) scan_u32_precleared_next();
    if ((st = scan_u32(w.hist, nullptr, w.hoff, hn, nullptr, hn, sp->counters + XG_CTR_ENTRIES,
                       bal ? scan2_ws : w.tail, bal ? scan2_bytes : w.tail_bytes, s)) != XG_OK)
      return st;
    const bool fused_order = sp->tile_order && n_tiles <= 1024;
    if (fused_order) {
      k_bin_ranges_order<<<1, 1024, 0, s>>>(w.hoff, C, n_tiles, sp->counters, cap, (long long*)sp->tile_ranges,
                                            sp->tile_order);
      if ((st = check_launch("k_bin_ranges_order")) != XG_OK) return st;
    } else {
      k_bin_ranges<<<div_up(n_tiles, 256), 256, 0, s>>>(w.hoff, C, n_tiles, sp->counters, cap,
                                                        (long long*)sp->tile_ranges);
      if ((st = check_launch("k_bin_ranges")) != XG_OK) return st;
    }
    if (bin_stop == 2) return XG_OK;
    if (bal) {
      const size_t sm_bal = sizeof(uint32_t) * ((size_t)n_tiles + (size_t)kBinWarps * ((n_tiles + 1) / 2));
      k_bin_emit_bal<<<C, kBinThreads, sm_bal, s>>>(sp->order, sp->n_tiles, (const ushort4*)sp->rect, w.offN, n, ntx,
                                                    n_tiles, sp->counters + XG_CTR_ENTRIES, w.hoff, w.wcnt, w.wstart,
                                                    cap, sp->entry_splat);
      if ((st = check_launch("k_bin_emit_bal")) != XG_OK) return st;
    } else {
      k_bin_emit<<<C, kBinThreads, sm_emit, s>>>(sp->order, sp->n_tiles, (const ushort4*)sp->rect, n, ntx, n_tiles,
                                                 rounds, w.hoff, w.wcnt, cap, sp->entry_splat);
      if ((st = check_launch("k_bin_emit")) != XG_OK) return st;
    }
    if (!sp->tile_order || fused_order) return XG_OK;
    return launch_tile_order(sp->tile_ranges, n_tiles, sp->tile_order, s);
  }
  // 2. offsets of every Gaussian's entries, in depth order
  if ((st = scan_u32(sp->n_tiles, sp->order, w.offN, n, nullptr, n, sp->counters + XG_CTR_ENTRIES,
                     w.tail, w.tail_bytes, s)) != XG_OK)
    return st;
  // 3. duplicate
  k_duplicate<<<div_up(n, 256), 256, 0, s>>>(sp->order, sp->n_tiles, (const ushort4*)sp->rect, w.offN,
                                             n, ntx, cap, w.keyE0, sp->entry_splat, sp->counters);
  if ((st = check_launch("k_duplicate")) != XG_OK) return st;
  // 4. stable sort by tile id
  int tile_bits = 0;
  while ((1 << tile_bits) < n_tiles) ++tile_bits;
  uint32_t* keys[2] = {w.keyE0, w.keyE1};
  uint32_t* vals[2] = {sp->entry_splat, w.valE1};
  int res = 0;
  if (tile_bits > 0) {
    if ((st = radix_sort_pairs(keys, vals, cap, sp->counters + XG_CTR_ENTRIES, 0, tile_bits, w.tail,
                               w.tail_bytes, s, &res)) != XG_OK)
      return st;
  }
  if (res == 1)
    cudaMemcpyAsync(sp->entry_splat, w.valE1, sizeof(uint32_t) * cap, cudaMemcpyDeviceToDevice, s);
  // 5. ranges
  cudaMemsetAsync(sp->tile_ranges, 0xff, sizeof(int64_t) * 2 * (size_t)n_tiles, s);
  k_tile_bounds<<<4 * 148, 256, 0, s>>>(keys[res], sp->counters, cap, (long long*)sp->tile_ranges);
  if ((st = check_launch("k_tile_bounds")) != XG_OK) return st;
  k_tile_fill<<<1, 1024, 0, s>>>(sp->counters, cap, n_tiles, (long long*)sp->tile_ranges);
  if ((st = check_launch("k_tile_fill")) != XG_OK) return st;
  if (!sp->tile_order) return XG_OK;
  return launch_tile_order(sp->tile_ranges, n_tiles, sp->tile_order, s);
}

}  // extern "C"
