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
#include "xg_sort.cuh"

namespace xg {
namespace {

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

__global__ void k_iota(uint32_t* v, long long n, uint32_t* n_dev) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
  if (i == 0) *n_dev = (uint32_t)n;
}

__global__ void k_duplicate(const uint32_t* __restrict__ order, const uint32_t* __restrict__ n_tiles,
                            const ushort4* __restrict__ rect, const uint32_t* __restrict__ offsets,
                            long long n, int ntx, long long cap, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals, uint32_t* counters) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool overflow = false;
  if (s < n) {
    const uint32_t g = order[s];
    const uint32_t cnt = n_tiles[g];
    if (cnt) {
      const long long off = offsets[s];
      if (off + cnt > cap) {
        overflow = true;
      } else {
        const ushort4 r = rect[g];
        long long o = off;
        for (int ty = r.y; ty <= r.w; ++ty)
          for (int tx = r.x; tx <= r.z; ++tx, ++o) {
            keys[o] = (uint32_t)(ty * ntx + tx);
            vals[o] = g;
          }
      }
    }
  }
  if (__ballot_sync(0xffffffffu, overflow) && lane_id() == 0)
    atomicOr(&counters[XG_CTR_STATUS], XG_ST_ENTRY_OVERFLOW);
}

__device__ __forceinline__ long long lower_bound(const uint32_t* a, long long n, uint32_t v) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_tile_ranges(const uint32_t* __restrict__ keys, const uint32_t* counters,
                              long long cap, int n_tiles, long long* __restrict__ ranges) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  long long e = counters[XG_CTR_ENTRIES];
  if (e > cap) e = cap;
  ranges[2 * t] = lower_bound(keys, e, (uint32_t)t);
  ranges[2 * t + 1] = lower_bound(keys, e, (uint32_t)t + 1);
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
  k_duplicate<<<div_up(n, 128), 128, 0, s>>>(sp->order, sp->n_tiles, (const ushort4*)sp->rect, w.offN,
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
  k_tile_ranges<<<div_up(n_tiles, 256), 256, 0, s>>>(keys[res], sp->counters, cap, n_tiles,
                                                      (long long*)sp->tile_ranges);
  if ((st = check_launch("k_tile_ranges")) != XG_OK) return st;
  if (!sp->tile_order) return XG_OK;
  return launch_tile_order(sp->tile_ranges, n_tiles, sp->tile_order, s);
}

}  // extern "C"
