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
  if (e > cap) e = cap;
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
  if (e > cap) e = cap;
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

struct BinWs {
  unsigned long long* keyN1;
  uint32_t *valN1, *offN, *keyE0, *keyE1, *valE1;
  void* tail;
  size_t tail_bytes;
};

size_t tail_bytes(int64_t n, int64_t cap) {
  size_t a = radix_workspace_bytes(n > cap ? n : cap);
  size_t b = scan_workspace_bytes(n);
  return a > b ? a : b;
}

bool carve(void* ws, size_t bytes, int64_t n, int64_t cap, BinWs& w) {
  char* p = (char*)ws;
  const size_t bn = align_up(sizeof(uint32_t) * (size_t)n);
  const size_t be = align_up(sizeof(uint32_t) * (size_t)(cap > 0 ? cap : 1));
  w.keyN1 = (unsigned long long*)p; p += 2 * bn;
  w.valN1 = (uint32_t*)p; p += bn;
  w.offN = (uint32_t*)p; p += bn;
  w.keyE0 = (uint32_t*)p; p += be;
  w.keyE1 = (uint32_t*)p; p += be;
  w.valE1 = (uint32_t*)p; p += be;
  w.tail = p;
  const size_t used = (size_t)(p - (char*)ws);
  const size_t tb = tail_bytes(n, cap);
  if (used + tb > bytes) return false;
  w.tail_bytes = bytes - used;
  return true;
}

}  // namespace
}  // namespace xg

using namespace xg;

extern "C" {

size_t xg_bin_workspace_bytes(int64_t n, int64_t entry_capacity, int32_t n_tiles_total) {
  (void)n_tiles_total;
  const size_t bn = align_up(sizeof(uint32_t) * (size_t)n);
  const size_t be = align_up(sizeof(uint32_t) * (size_t)(entry_capacity > 0 ? entry_capacity : 1));
  return 4 * bn + 3 * be + tail_bytes(n, entry_capacity) + 256;
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
  if (!carve(workspace, workspace_bytes, n, cap, w)) {
    set_error_msg("xg_bin_sort: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int ntx = tiles_x(*cam), nty = tiles_y(*cam);
  const int n_tiles = ntx * nty;
  xg_status st;
  // n as a device count for the generic sort: stash it in counters[TOUCH]
  uint32_t* n_dev = sp->counters + XG_CTR_TOUCH;
  // 1. depth sort
  k_iota<<<div_up(n, 256), 256, 0, s>>>(sp->order, n, n_dev);
  if ((st = check_launch("k_iota")) != XG_OK) return st;
  {
    unsigned long long* keys[2] = {(unsigned long long*)sp->depth_key, w.keyN1};
    uint32_t* vals[2] = {sp->order, w.valN1};
    int res = 0;
    if ((st = radix_sort_pairs64(keys, vals, n, n_dev, 0, 64, w.tail, w.tail_bytes, s, &res)) != XG_OK)
      return st;
    if (res == 1) cudaMemcpyAsync(sp->order, w.valN1, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s);
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
