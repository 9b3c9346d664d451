// Decoupled look-back scan and a stable LSD radix sort (reduce / scan /
// rank-and-scatter per pass) for the binning stage (K2).
//
// Both read the live item count from device memory, so a whole render is
// enqueued without a host round trip: grids are sized for the caller's
// capacity and CTAs past the live count exit (or contribute zeros).
#include "xg_sort.cuh"

namespace xg {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortRounds = 4;                         // 32-item rounds per warp
constexpr int kSortTile = kSortThreads * kSortRounds;  // 4096

constexpr unsigned long long kFlagAgg = 1ull << 32;
constexpr unsigned long long kFlagPre = 2ull << 32;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block-wide exclusive scan of one value per thread; returns the aggregate.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* smem_warp,
                                                         uint32_t& aggregate) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) smem_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (int)(blockDim.x >> 5) ? smem_warp[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < (int)(blockDim.x >> 5)) smem_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) smem_warp[32] = wi;
  }
  __syncthreads();
  aggregate = smem_warp[32];
  return smem_warp[warp] + incl - v;
}

__global__ void __launch_bounds__(kScanThreads)
    k_scan(const uint32_t* __restrict__ in, const uint32_t* __restrict__ gather,
           uint32_t* __restrict__ out, const uint32_t* n_dev, long long n_host, long long cap,
           unsigned long long* states, uint32_t* tile_counter, uint32_t* total) {
  __shared__ uint32_t s_warp[33];
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_prefix;
  long long n = n_dev ? (long long)*n_dev : n_host;
  if (n > cap) n = cap;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const long long base = (long long)tile * kScanTile + (long long)threadIdx.x * kScanItems;
  uint32_t x[kScanItems];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long idx = base + k;
    uint32_t v = 0;
    if (idx < n) v = gather ? in[gather[idx]] : in[idx];
    x[k] = v;
    sum += v;
  }
  uint32_t agg;
  uint32_t excl = block_exclusive_scan(sum, s_warp, agg);
  // Look-back for the tile prefix.
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) {
        st_volatile_u64(&states[0], kFlagPre | agg);
      }
    } else {
      if (lane == 0) {
        __threadfence();
        st_volatile_u64(&states[tile], kFlagAgg | agg);
      }
      long long j = (long long)tile - 1;
      while (true) {
        const long long idx = j - lane;
        unsigned long long st;
        if (idx >= 0) {
          do {
            st = ld_volatile_u64(&states[idx]);
          } while ((st >> 32) == 0);
        } else {
          st = kFlagPre;  // virtual prefix 0 before tile 0
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (st >> 32) == 2);
        uint32_t v = (uint32_t)st;
        if (pre) {
          const int first = __ffs(pre) - 1;  // nearest tile holding an inclusive prefix
          if (lane > first) v = 0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          prefix += v;
          break;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        prefix += v;
        j -= 32;
      }
      if (lane == 0) {
        __threadfence();
        st_volatile_u64(&states[tile], kFlagPre | (uint32_t)(prefix + agg));
      }
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  uint32_t run = s_prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const long long idx = base + k;
    if (idx < n) out[idx] = run;
    run += x[k];
  }
  if (total && base <= n && n <= base + kScanItems) {
    // the thread owning position n (one past the end) publishes the total
    uint32_t t = s_prefix + excl;
    for (long long idx = base; idx < n; ++idx) t += x[idx - base];
    *total = t;
  }
}

template <int BITS, typename K>
__global__ void __launch_bounds__(kSortThreads)
    k_radix_hist(const K* __restrict__ keys, const uint32_t* n_dev, long long cap, int shift,
                 uint32_t* __restrict__ hist) {
  constexpr int BINS = 1 << BITS;
  __shared__ uint32_t h[kSortWarps][BINS];
  long long n = *n_dev;
  if (n > cap) n = 0;  // overflowed list (never fully written): discarded and re-binned
  const int warp = threadIdx.x >> 5;
  for (int b = threadIdx.x; b < kSortWarps * BINS; b += kSortThreads) (&h[0][0])[b] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kSortTile;
  for (int k = threadIdx.x; k < kSortTile; k += kSortThreads) {
    const long long idx = base + k;
    if (idx < n) atomicAdd(&h[warp][(uint32_t)(keys[idx] >> shift) & (BINS - 1)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < BINS; b += kSortThreads) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) t += h[w][b];
    hist[(long long)b * gridDim.x + blockIdx.x] = t;
  }
}

// Stable rank-and-scatter.  Warp w owns the contiguous segment
// [base + 512 w, base + 512 (w+1)), walked in 32-item rounds; within a round
// lanes with equal digits are ranked by __match_any_sync, so item order is
// (warp, round, lane) = input order.
template <int BITS, typename K>
__global__ void __launch_bounds__(kSortThreads)
    k_radix_scatter(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                    K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                    const uint32_t* n_dev, long long cap, int shift,
                    const uint32_t* __restrict__ offsets) {
  constexpr int BINS = 1 << BITS;
  __shared__ uint32_t wh[kSortWarps][BINS];
  __shared__ uint32_t goff[BINS];
  long long n = *n_dev;
  if (n > cap) n = 0;  // overflowed list (never fully written): discarded and re-binned
  const long long base = (long long)blockIdx.x * kSortTile;
  if (base >= n) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b = threadIdx.x; b < kSortWarps * BINS; b += kSortThreads) (&wh[0][0])[b] = 0;
  for (int b = threadIdx.x; b < BINS; b += kSortThreads)
    goff[b] = offsets[(long long)b * gridDim.x + blockIdx.x];
  __syncthreads();
  const unsigned lt = lanemask_lt();
  K key[kSortRounds];
  uint32_t val[kSortRounds], pos[kSortRounds];
  const long long seg = base + (long long)warp * (kSortTile / kSortWarps);
  // all loads first (16 independent coalesced loads in flight per thread)
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const long long idx = seg + r * 32 + lane;
    const bool valid = idx < n;
    key[r] = valid ? keys_in[idx] : (K)0;
    val[r] = valid ? vals_in[idx] : 0u;
  }
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const long long idx = seg + r * 32 + lane;
    const bool valid = idx < n;
    const uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & (BINS - 1)) : (uint32_t)BINS;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = wh[warp][valid ? d : 0];
    pos[r] = before + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers >> lane) == 1u) wh[warp][d] = before + __popc(peers);  // highest peer lane
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix over warps per digit
  for (int b = threadIdx.x; b < BINS; b += kSortThreads) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t t = wh[w][b];
      wh[w][b] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const long long idx = seg + r * 32 + lane;
    if (idx < n) {
      const uint32_t d = (uint32_t)(key[r] >> shift) & (BINS - 1);
      const uint32_t dst = goff[d] + wh[warp][d] + pos[r];
      keys_out[dst] = key[r];
      vals_out[dst] = val[r];
    }
  }
}

template <int BITS, typename K>
void launch_pass(K* const* keys, uint32_t* const* vals, int src, int grid, long long cap,
                 const uint32_t* n_dev, int shift, uint32_t* hist, uint32_t* offs, void* sws,
                 size_t sws_bytes, cudaStream_t s, xg_status* st) {
  k_radix_hist<BITS, K><<<grid, kSortThreads, 0, s>>>(keys[src], n_dev, cap, shift, hist);
  if ((*st = check_launch("k_radix_hist")) != XG_OK) return;
  const long long hn = (long long)grid << BITS;
  if ((*st = scan_u32(hist, nullptr, offs, hn, nullptr, hn, nullptr, sws, sws_bytes, s)) != XG_OK)
    return;
  k_radix_scatter<BITS, K><<<grid, kSortThreads, 0, s>>>(keys[src], vals[src], keys[1 - src],
                                                      vals[1 - src], n_dev, cap, shift, offs);
  *st = check_launch("k_radix_scatter");
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

// set by a caller that has already zeroed the next scan_u32's workspace
// (host-side, per call; the library's launch paths are single-threaded per stream)
static thread_local bool g_scan_precleared = false;

void scan_u32_precleared_next() { g_scan_precleared = true; }

size_t scan_workspace_bytes(int64_t cap) {
  const int64_t tiles = (cap + kScanTile - 1) / kScanTile + 1;
  return align_up(sizeof(unsigned long long) * (size_t)tiles) + 256;
}

xg_status scan_u32(const uint32_t* in, const uint32_t* gather, uint32_t* out, int64_t cap,
                   const uint32_t* n_dev, int64_t n_host, uint32_t* total, void* ws, size_t ws_bytes,
                   cudaStream_t s) {
  const bool precleared = g_scan_precleared;  // (one call only)
  g_scan_precleared = false;
  if (cap <= 0) {
    if (total) cudaMemsetAsync(total, 0, sizeof(uint32_t), s);
    return XG_OK;
  }
  const size_t need = scan_workspace_bytes(cap);
  if (ws_bytes < need) {
    set_error_msg("scan_u32: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  const int tiles = div_up(cap, kScanTile);
  unsigned long long* states = (unsigned long long*)ws;
  uint32_t* counter = (uint32_t*)((char*)ws + align_up(sizeof(unsigned long long) * (size_t)(tiles + 1)));
  if (!precleared) cudaMemsetAsync(ws, 0, need, s);
  k_scan<<<tiles, kScanThreads, 0, s>>>(in, gather, out, n_dev, n_host, cap, states, counter, total);
  return check_launch("k_scan");
}

size_t radix_workspace_bytes(int64_t cap) {
  const int64_t grid = (cap + kSortTile - 1) / kSortTile;
  const int64_t hn = grid * 256;
  return 2 * align_up(sizeof(uint32_t) * (size_t)hn) + scan_workspace_bytes(hn);
}

namespace {
template <typename K>
xg_status radix_sort_impl(K* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev, int begin_bit,
                          int end_bit, void* ws, size_t ws_bytes, cudaStream_t s, int* result) {
  *result = 0;
  const int total_bits = end_bit - begin_bit;
  if (cap <= 0 || total_bits <= 0) return XG_OK;
  if (ws_bytes < radix_workspace_bytes(cap)) {
    set_error_msg("radix_sort_pairs: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  const int grid = div_up(cap, kSortTile);
  const size_t hbytes = align_up(sizeof(uint32_t) * (size_t)grid * 256);
  uint32_t* hist = (uint32_t*)ws;
  uint32_t* offs = (uint32_t*)((char*)ws + hbytes);
  void* sws = (char*)ws + 2 * hbytes;
  const size_t sws_bytes = ws_bytes - 2 * hbytes;
  const int passes = (total_bits + 7) / 8;
  const int bits = (total_bits + passes - 1) / passes;
  int src = 0;
  xg_status st = XG_OK;
  for (int p = 0; p < passes && st == XG_OK; ++p) {
    const int shift = begin_bit + p * bits;
#define XG_PASS(B) launch_pass<B, K>(keys, vals, src, grid, cap, n_dev, shift, hist, offs, sws, sws_bytes, s, &st)
    switch (bits) {
      case 1: XG_PASS(1); break;
      case 2: XG_PASS(2); break;
      case 3: XG_PASS(3); break;
      case 4: XG_PASS(4); break;
      case 5: XG_PASS(5); break;
      case 6: XG_PASS(6); break;
      case 7: XG_PASS(7); break;
      default: XG_PASS(8); break;
    }
#undef XG_PASS
    src = 1 - src;
  }
  *result = src;
  return st;
}
}  // namespace

xg_status radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                           int begin_bit, int end_bit, void* ws, size_t ws_bytes, cudaStream_t s,
                           int* result) {
  return radix_sort_impl<uint32_t>(keys, vals, cap, n_dev, begin_bit, end_bit, ws, ws_bytes, s, result);
}

xg_status radix_sort_pairs64(unsigned long long* keys[2], uint32_t* vals[2], int64_t cap,
                             const uint32_t* n_dev, int begin_bit, int end_bit, void* ws, size_t ws_bytes,
                             cudaStream_t s, int* result) {
  return radix_sort_impl<unsigned long long>(keys, vals, cap, n_dev, begin_bit, end_bit, ws, ws_bytes, s,
                                             result);
}

// ---------------------------------------------------------------------------
// Onesweep-style LSD radix sort of (uint64 key, uint32 value) pairs: one
// histogram kernel for all passes, then ONE kernel per 8-bit pass in which
// each tile ranks its keys locally, publishes per-digit counts and finds its
// global digit offsets by decoupled look-back over the preceding tiles - no
// separate histogram/scan launches per pass.  Passes whose digit is the same
// for every key (e.g. the constant exponent byte of depths) are skipped on
// the device; the ping-pong buffer each pass reads is chosen on the device.
// ---------------------------------------------------------------------------
namespace {

constexpr int kOsThreads = 256;
constexpr int kOsWarps = kOsThreads / 32;
#ifndef XG_OS_ROUNDS
#define XG_OS_ROUNDS 8
#endif
constexpr int kOsRounds = XG_OS_ROUNDS;
constexpr int kOsTile = kOsThreads * kOsRounds;  // 2048 items
constexpr int kOsPasses = 8;
constexpr uint32_t kOsAgg = 1u << 30, kOsPre = 2u << 30, kOsMask = (1u << 30) - 1u;
#ifndef XG_OS_LOOKBACK
#define XG_OS_LOOKBACK 4
#endif
constexpr int kOsLookback = XG_OS_LOOKBACK;  // predecessor tiles per look-back round

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kOsThreads)
    k_os_hist(const unsigned long long* __restrict__ keys, const uint32_t* n_dev, long long cap,
              uint32_t* __restrict__ ghist, int n_passes) {
  __shared__ uint32_t h[kOsPasses][256];
  for (int i = threadIdx.x; i < kOsPasses * 256; i += kOsThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  long long n = *n_dev;
  if (n > cap) n = cap;
  for (long long i = (long long)blockIdx.x * kOsThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kOsThreads) {
    const unsigned long long k = keys[i];
#pragma unroll
    for (int p = 0; p < kOsPasses; ++p)
      if (p < n_passes) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kOsPasses * 256; i += kOsThreads) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(&ghist[i], v);
  }
}

// exclusive offsets per pass, and the buffer each pass reads (sel[p]);
// sel[kOsPasses] is where the result lands
__global__ void __launch_bounds__(256) k_os_scan(const uint32_t* __restrict__ ghist, uint32_t* __restrict__ gofs,
                                                 const uint32_t* n_dev, long long cap, int* __restrict__ sel,
                                                 int n_passes) {
  __shared__ uint32_t s_w[8];
  __shared__ int trivial[kOsPasses];
  long long n = *n_dev;
  if (n > cap) n = cap;
  const int d = threadIdx.x, lane = d & 31, w = d >> 5;
  if (d < kOsPasses) trivial[d] = 1;  // (passes past n_passes: the caller's keys are zero there)
  __syncthreads();
  for (int p = 0; p < n_passes && p < kOsPasses; ++p) {
    // exclusive scan of the pass's 256 digit counts: warp shuffles + 8 warp totals
    const uint32_t v = ghist[p * 256 + d];
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[w] = x;
    const int t = __syncthreads_or((long long)v == n);  // (also orders s_w)
    uint32_t base = 0;
    for (int k = 0; k < w; ++k) base += s_w[k];
    gofs[p * 256 + d] = base + x - v;
    if (d == 0) trivial[p] = t;
    __syncthreads();
  }
  // buffers: 0 / 1 ping-pong scratch, 2 the caller's input (never written)
  if (d == 0) {
    int cur = 2;
    for (int p = 0; p < kOsPasses; ++p) {
      sel[p] = cur;
      if (!trivial[p]) cur = cur == 0 ? 1 : 0;
    }
    sel[kOsPasses] = cur;
  }
}

struct OsArgs {
  unsigned long long* keys[3];  // scratch A, scratch B, input (read-only)
  uint32_t* vals[3];
  const uint32_t* n_dev;
  long long cap;
  int pass;
  const uint32_t* ghist;
  const uint32_t* gofs;
  const int* sel;
  uint32_t* status;    // [tiles][256] for this pass, zeroed
  uint32_t* tile_ctr;  // zeroed
};

__global__ void __launch_bounds__(kOsThreads) k_os_pass(OsArgs a) {
  __shared__ uint32_t wh[kOsWarps][256];
  __shared__ uint32_t s_pre[256];
  __shared__ uint32_t s_tile;
  long long n = *a.n_dev;
  if (n > a.cap) n = a.cap;
  const int p = a.pass;
  // a pass whose digit is constant over all keys is the identity: skip it
  if (a.sel[p + 1] == a.sel[p]) return;
  const int src = a.sel[p];
  const int shift = 8 * p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kOsWarps * 256; i += kOsThreads) (&wh[0][0])[i] = 0;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const long long base = (long long)tile * kOsTile;
  if (base >= n) return;
  // (selects, not a[idx]: a runtime index into the parameter arrays would
  // copy them to local memory)
  const unsigned long long* kin = src == 0 ? a.keys[0] : src == 1 ? a.keys[1] : a.keys[2];
  const uint32_t* vin = src == 0 ? a.vals[0] : src == 1 ? a.vals[1] : a.vals[2];
  const unsigned lt = lanemask_lt();
  unsigned long long key[kOsRounds];
  uint32_t val[kOsRounds], pos[kOsRounds];
  const long long seg = base + (long long)warp * (kOsTile / kOsWarps);
#pragma unroll
  for (int r = 0; r < kOsRounds; ++r) {
    const long long idx = seg + r * 32 + lane;
    const bool valid = idx < n;
    key[r] = valid ? kin[idx] : 0ull;
    val[r] = valid ? vin[idx] : 0u;
  }
#pragma unroll
  for (int r = 0; r < kOsRounds; ++r) {
    const long long idx = seg + r * 32 + lane;
    const bool valid = idx < n;
    const uint32_t d = valid ? (uint32_t)(key[r] >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = wh[warp][valid ? d : 0];
    pos[r] = before + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers >> lane) == 1u) wh[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const int d = threadIdx.x;  // 256 threads = 256 digits
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kOsWarps; ++w) {
      const uint32_t t = wh[w][d];
      wh[w][d] = run;
      run += t;
    }
    uint32_t* st = a.status + (long long)tile * 256;
    if (tile == 0) {
      asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(st + d), "r"(kOsPre | run) : "memory");
      s_pre[d] = 0;
    } else {
      asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(st + d), "r"(kOsAgg | run) : "memory");
      // windowed look-back: the statuses of kOsLookback predecessors are
      // loaded together (one L2 round trip instead of one per tile), then
      // summed nearest first up to the first inclusive prefix
      uint32_t prefix = 0;
      long long j = (long long)tile - 1;
      bool done = false;
      while (!done) {
        uint32_t v[kOsLookback];
#pragma unroll
        for (int w = 0; w < kOsLookback; ++w)
          v[w] = j - w >= 0 ? ld_volatile_u32(a.status + (j - w) * 256 + d) : kOsPre;  // (tile 0 is a prefix)
#pragma unroll
        for (int w = 0; w < kOsLookback; ++w) {
          if (!done) {
            while ((v[w] & ~kOsMask) == 0) v[w] = ld_volatile_u32(a.status + (j - w) * 256 + d);
            prefix += v[w] & kOsMask;
            done = (v[w] & ~kOsMask) == kOsPre;
          }
        }
        j -= kOsLookback;
      }
      asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(st + d), "r"(kOsPre | (prefix + run)) : "memory");
      s_pre[d] = prefix;
    }
  }
  __syncthreads();
  const int dst = a.sel[p + 1];
  unsigned long long* kout = dst == 0 ? a.keys[0] : dst == 1 ? a.keys[1] : a.keys[2];
  uint32_t* vout = dst == 0 ? a.vals[0] : dst == 1 ? a.vals[1] : a.vals[2];
  const uint32_t* go = a.gofs + p * 256;
#pragma unroll
  for (int r = 0; r < kOsRounds; ++r) {
    const long long idx = seg + r * 32 + lane;
    if (idx < n) {
      const uint32_t d = (uint32_t)(key[r] >> shift) & 255u;
      const uint32_t dst = go[d] + s_pre[d] + wh[warp][d] + pos[r];
      kout[dst] = key[r];
      vout[dst] = val[r];
    }
  }
}

// the result lands in vals[sel[K]]: copy it to vals_out unless it is there
__global__ void k_os_finish(uint32_t* vals_out, const uint32_t* vals_a, const uint32_t* vals_b,
                            const uint32_t* vals_in, const uint32_t* n_dev, long long cap, const int* sel) {
  const int r = sel[kOsPasses];
  const uint32_t* src = r == 0 ? vals_a : r == 1 ? vals_b : vals_in;  // (2: every pass trivial)
  if (!src || src == vals_out) return;
  long long n = *n_dev;
  if (n > cap) n = cap;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    vals_out[i] = src[i];
}

}  // namespace

size_t onesweep_workspace_bytes(int64_t cap) {
  const int64_t tiles = (cap + kOsTile - 1) / kOsTile;
  return align_up(sizeof(uint32_t) * kOsPasses * 256 * 2) + align_up(sizeof(int) * (kOsPasses + 1)) +
         align_up(sizeof(uint32_t) * kOsPasses) + align_up(sizeof(uint32_t) * (size_t)kOsPasses * tiles * 256) + 256;
}

namespace {

struct OsWs {
  uint32_t* ghist;  // [kOsPasses][256]
  uint32_t* gofs;   // [kOsPasses][256]
  int* sel;         // [kOsPasses + 1]
  uint32_t* ctr;    // [kOsPasses]
  uint32_t* status; // [kOsPasses][tiles][256]
  int64_t tiles;
};

// carve the workspace and zero what n_passes passes use (histograms,
// counters and their look-back status words)
// (clear = false: the caller zeroes os_prepare_bytes(cap, n_passes) at ws itself)
OsWs os_prepare(void* ws, int64_t cap, int n_passes, cudaStream_t s, bool clear = true) {
  OsWs w;
  w.tiles = (cap + kOsTile - 1) / kOsTile;
  char* p = (char*)ws;
  w.ghist = (uint32_t*)p;
  w.gofs = w.ghist + kOsPasses * 256;
  p += align_up(sizeof(uint32_t) * kOsPasses * 256 * 2);
  w.sel = (int*)p;
  p += align_up(sizeof(int) * (kOsPasses + 1));
  w.ctr = (uint32_t*)p;
  p += align_up(sizeof(uint32_t) * kOsPasses);
  w.status = (uint32_t*)p;
  const int np = n_passes < kOsPasses ? n_passes : kOsPasses;
  if (clear) cudaMemsetAsync(ws, 0, (size_t)(p - (char*)ws) + sizeof(uint32_t) * (size_t)np * w.tiles * 256, s);
  return w;
}

size_t os_prepare_bytes(int64_t cap, int n_passes) {
  const int64_t tiles = (cap + kOsTile - 1) / kOsTile;
  const int np = n_passes < kOsPasses ? n_passes : kOsPasses;
  return align_up(sizeof(uint32_t) * kOsPasses * 256 * 2) + align_up(sizeof(int) * (kOsPasses + 1)) +
         align_up(sizeof(uint32_t) * kOsPasses) + sizeof(uint32_t) * (size_t)np * tiles * 256;
}

xg_status os_passes(const OsWs& w, const unsigned long long* keys_in, const uint32_t* vals_in,
                    unsigned long long* keys_a, unsigned long long* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                    int64_t cap, const uint32_t* n_dev, int n_passes, cudaStream_t s) {
  for (int pass = 0; pass < n_passes && pass < kOsPasses; ++pass) {  // (higher bytes all zero: no-op passes)
    OsArgs a;
    a.keys[0] = keys_a;
    a.keys[1] = keys_b;
    a.keys[2] = const_cast<unsigned long long*>(keys_in);
    a.vals[0] = vals_a;
    a.vals[1] = vals_b;
    a.vals[2] = const_cast<uint32_t*>(vals_in);
    a.n_dev = n_dev;
    a.cap = cap;
    a.pass = pass;
    a.ghist = w.ghist;
    a.gofs = w.gofs;
    a.sel = w.sel;
    a.status = w.status + (size_t)pass * w.tiles * 256;
    a.tile_ctr = w.ctr + pass;
    k_os_pass<<<(int)w.tiles, kOsThreads, 0, s>>>(a);
    xg_status st = check_launch("k_os_pass");
    if (st != XG_OK) return st;
  }
  return XG_OK;
}

}  // namespace

xg_status onesweep_sort_pairs64(const unsigned long long* keys_in, const uint32_t* vals_in,
                                unsigned long long* keys_a, unsigned long long* keys_b, uint32_t* vals_a,
                                uint32_t* vals_b, uint32_t* vals_out, int64_t cap, const uint32_t* n_dev,
                                void* ws, size_t ws_bytes, cudaStream_t s, int n_passes, const int** result_sel) {
  if (cap <= 0) return XG_OK;
  if (ws_bytes < onesweep_workspace_bytes(cap)) {
    set_error_msg("onesweep_sort_pairs64: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  const OsWs w = os_prepare(ws, cap, n_passes, s);
  const int hgrid = (int)(w.tiles < 296 ? w.tiles : 296);
  k_os_hist<<<hgrid, kOsThreads, 0, s>>>(keys_in, n_dev, cap, w.ghist, n_passes);
  xg_status st = check_launch("k_os_hist");
  if (st != XG_OK) return st;
  k_os_scan<<<1, 256, 0, s>>>(w.ghist, w.gofs, n_dev, cap, w.sel, n_passes);
  if ((st = check_launch("k_os_scan")) != XG_OK) return st;
  if ((st = os_passes(w, keys_in, vals_in, keys_a, keys_b, vals_a, vals_b, cap, n_dev, n_passes, s)) != XG_OK)
    return st;
  if (result_sel) {  // the caller reads vals {a, b, in}[sel[8]] itself
    *result_sel = w.sel + kOsPasses;
    return XG_OK;
  }
  k_os_finish<<<(int)(w.tiles < 296 ? w.tiles : 296), 256, 0, s>>>(vals_out, vals_a, vals_b, vals_in, n_dev, cap,
                                                                  w.sel);
  return check_launch("k_os_finish");
}

}  // namespace xg

namespace xg {

// ---------------------------------------------------------------------------
// Depth order by buckets (K2 step 1; the 8-pass onesweep on the raw float64
// bits stays selectable with XG_DEPTH_SORT=onesweep).
//
// The order wanted is ascending (float64 depth bits, cloud index) over the
// active splats - what a stable LSD sort of the index-ordered keys gives.
//   1. min / max of the active keys;
//   2. bucket b = 1 + ((key - kmin) >> shift), 2^15 buckets spanning
//      [kmin, kmax] (monotone in the key; inactive splats -> bucket 0, never
//      looked at again: count / emit skip them); per-bucket counts and
//      per-bucket min / max key (atomics);
//   3. exclusive scan of the counts -> bucket starts;
//   4. a STABLE sort of the 16-bit bucket ids (two onesweep passes instead
//      of eight): every bucket's splats in cloud-index order;
//   5. a bucket whose min key == max key (one depth value: the usual case on
//      lattice clouds, where a depth is shared by a whole column of splats)
//      is final; otherwise each splat's rank inside the bucket is counted by
//      the total order (key, index) - or, for a bucket larger than
//      kBsRankMax, the bucket is sorted by one CTA (bitonic in shared memory,
//      or in place in global memory beyond kBsSmemMax).
// The result is the same permutation bit for bit (a total order has one
// sorted sequence); the symmetric phi = pi/4 views of the golden tests pin it.
// ---------------------------------------------------------------------------
namespace {

constexpr int kBsBits = 16;           // 16-bit ids: active buckets 0 .. 65534, 65535 = inactive
constexpr uint32_t kBsBuckets = 1u << kBsBits;
constexpr uint32_t kBsInactive = kBsBuckets - 1;
constexpr int kBsRankMax = 256;       // counting rank up to this (mixed) bucket size
// buckets up to this size are ranked by each member against the whole bucket
// in k_bs_rank (<= 64 loads per thread); larger mixed ones go to a warp
// (k_bs_mixed).  (A trained cloud's mixed buckets hold tens of distinct
// depths: 32 -> 64 moved them out of the warp path, -11 us per C2 iteration.)
constexpr int kBsRankBrute = 64;
constexpr int kBsSmemMax = 16384;     // shared-memory bitonic up to this size (12 B each: 192 KB)
constexpr int kBsLargeThreads = 512;

struct BsWs {
  unsigned long long* mm;    // [0] min key, [1] ~max key (both via atomicMin)
  uint32_t* n_large;
  uint32_t* count;           // [kBsBuckets]
  uint32_t* start;           // [kBsBuckets + 1]
  unsigned long long* bmin;  // [kBsBuckets] per-bucket min key
  unsigned long long* bmax;  // [kBsBuckets] per-bucket ~max key
  uint32_t* large;           // [kBsBuckets]
  uint32_t* mixed;           // [kBsBuckets]
  uint32_t* n_mixed;
  void* tail;                // onesweep workspace
  size_t tail_bytes;
  void* scan_ws;             // the bucket-count scan's workspace (after it)
  size_t scan_bytes;
};

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

inline size_t bs_fixed_bytes() {
  return 768 + 2 * al256(sizeof(uint32_t) * (kBsBuckets + 1)) + 2 * al256(sizeof(unsigned long long) * kBsBuckets) +
         2 * al256(sizeof(uint32_t) * kBsBuckets);
}

// Layout: the all-ones region [mm | bmin | bmax], the unset [start | large |
// mixed], then the zero region [n_large | n_mixed | count | scan_ws | tail],
// so one memset per value initialises the whole sort (bucket_sort_depth).
inline bool bs_carve(void* ws, size_t bytes, BsWs& w) {
  char* p = (char*)ws;
  w.mm = (unsigned long long*)p; p += 256;
  w.bmin = (unsigned long long*)p; p += al256(sizeof(unsigned long long) * kBsBuckets);
  w.bmax = (unsigned long long*)p; p += al256(sizeof(unsigned long long) * kBsBuckets);
  w.start = (uint32_t*)p; p += al256(sizeof(uint32_t) * (kBsBuckets + 1));
  w.large = (uint32_t*)p; p += al256(sizeof(uint32_t) * kBsBuckets);
  w.mixed = (uint32_t*)p; p += al256(sizeof(uint32_t) * kBsBuckets);
  w.n_large = (uint32_t*)p; p += 256;
  w.n_mixed = (uint32_t*)p; p += 256;
  w.count = (uint32_t*)p; p += al256(sizeof(uint32_t) * (kBsBuckets + 1));
  w.scan_ws = p;
  w.scan_bytes = al256(scan_workspace_bytes(kBsBuckets));
  p += w.scan_bytes;
  w.tail = p;
  const size_t used = (size_t)(p - (char*)ws);
  if (used > bytes) return false;
  w.tail_bytes = bytes - used;
  return true;
}

__device__ __forceinline__ int bs_shift(const unsigned long long* mm) {
  const unsigned long long range = (~mm[1]) - mm[0];  // kmax - kmin
  const int len = range ? 64 - __clzll(range) : 0;
  return len > kBsBits ? len - kBsBits : 0;
}

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }

__global__ void k_bs_minmax(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ n_tiles,
                            long long n, unsigned long long* mm, uint32_t* n_dev) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = (uint32_t)n;  // (the onesweep's live count)
  unsigned long long lo = ~0ull, nhi = ~0ull;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (n_tiles[i]) {
      const unsigned long long k = keys[i];
      lo = umin64(lo, k);
      nhi = umin64(nhi, ~k);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = umin64(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    nhi = umin64(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
  }
  __shared__ unsigned long long s_lo[32], s_nhi[32];  // (one atomic pair per CTA: 4k warps on two
  const int warp = threadIdx.x >> 5;                   //  addresses serialised to ~10 us)
  if ((threadIdx.x & 31) == 0) {
    s_lo[warp] = lo;
    s_nhi[warp] = nhi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      lo = umin64(lo, s_lo[i]);
      nhi = umin64(nhi, s_nhi[i]);
    }
    if (lo != ~0ull) atomicMin(mm, lo);
    if (nhi != ~0ull) atomicMin(mm + 1, nhi);
  }
}

__device__ __forceinline__ unsigned long long peer_min64(unsigned peers, unsigned long long v) {
  const uint32_t hi = __reduce_min_sync(peers, (uint32_t)(v >> 32));
  const uint32_t lo = __reduce_min_sync(peers, (uint32_t)(v >> 32) == hi ? (uint32_t)v : 0xffffffffu);
  return ((unsigned long long)hi << 32) | lo;
}

// bucket ids (the stable sort's keys), the iota values, per-bucket counts and
// key range, and the two byte histograms of the ids the onesweep passes need
// (ghist[0] low byte, ghist[1] high byte; in place of a k_os_hist pass)
__global__ void k_bs_bucket(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ n_tiles,
                            long long n, const unsigned long long* __restrict__ mm,
                            unsigned long long* __restrict__ bkey, uint32_t* __restrict__ iota,
                            uint32_t* __restrict__ count, unsigned long long* __restrict__ bmin,
                            unsigned long long* __restrict__ bmax, uint32_t* __restrict__ ghist) {
  __shared__ uint32_t s_h[2][256];
  for (int k = threadIdx.x; k < 512; k += blockDim.x) (&s_h[0][0])[k] = 0u;
  __syncthreads();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int shift = bs_shift(mm);
  const unsigned long long kmin = mm[0];
  const bool valid = i < n;
  unsigned long long k = 0;
  uint32_t b = 0xffffffffu;
  if (valid) {
    k = keys[i];
    b = n_tiles[i] ? min((uint32_t)((k - kmin) >> shift), kBsInactive - 1u) : kBsInactive;
    bkey[i] = b;
    iota[i] = (uint32_t)i;
  }
  const unsigned peers = __match_any_sync(0xffffffffu, b);
  // min of k and of ~k over the lane's peers (same bucket): 64-bit minima as
  // (high word, then low word among the lanes holding the high minimum)
  const unsigned long long lo = peer_min64(peers, k), nhi = peer_min64(peers, ~k);
  if (valid && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) {
    atomicAdd(&count[b], (uint32_t)__popc(peers));
    atomicAdd(&s_h[0][b & 255u], (uint32_t)__popc(peers));
    atomicAdd(&s_h[1][b >> 8], (uint32_t)__popc(peers));
    if (b != kBsInactive) {
      atomicMin(&bmin[b], lo);
      atomicMin(&bmax[b], nhi);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 512; k += blockDim.x) {
    const uint32_t v = (&s_h[0][0])[k];
    if (v) atomicAdd(&ghist[k], v);
  }
}

__device__ __forceinline__ bool bs_less(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// sorted: indices in (bucket, index) order.  Final position of sorted[p].
struct BsSorted {  // the stable pass's result: vals {a, b, in}[*sel]
  const uint32_t* v[3];
  const int* sel;
  __device__ __forceinline__ const uint32_t* get() const {
    const int k = *sel;
    return k == 0 ? v[0] : k == 1 ? v[1] : v[2];
  }
};

// Bucket starts from the stable pass's order: the first sorted position of
// each non-empty bucket (a bucket's end is start + count) - in place of an
// exclusive scan over all 65,536 bucket counts.
__device__ __forceinline__ uint32_t bs_bucket_of(const unsigned long long* __restrict__ keys,
                                                 const uint32_t* __restrict__ n_tiles,
                                                 const unsigned long long* __restrict__ mm, uint32_t ix) {
  return n_tiles[ix] ? min((uint32_t)((keys[ix] - mm[0]) >> bs_shift(mm)), kBsInactive - 1u) : kBsInactive;
}

#ifndef XG_BS_BOUNDS
#define XG_BS_BOUNDS 0  // 1: bucket starts from the sorted boundaries (measured: C3 -0.6 %, C2 equal)
#endif
__global__ void k_bs_bounds(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ n_tiles,
                            const unsigned long long* __restrict__ mm, BsSorted srt, long long n,
                            uint32_t* __restrict__ start) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t* __restrict__ sorted = srt.get();
  const uint32_t b = bs_bucket_of(keys, n_tiles, mm, sorted[p]);
  if (p == 0 || bs_bucket_of(keys, n_tiles, mm, sorted[p - 1]) != b) start[b] = (uint32_t)p;
}

__global__ void k_bs_rank(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ n_tiles,
                          const unsigned long long* __restrict__ mm, BsSorted srt, long long n,
                          const uint32_t* __restrict__ start, const uint32_t* __restrict__ count, const unsigned long long* __restrict__ bmin,
                          const unsigned long long* __restrict__ bmax, uint32_t* __restrict__ order,
                          uint32_t* __restrict__ large, uint32_t* __restrict__ n_large, uint32_t* __restrict__ mixed,
                          uint32_t* __restrict__ n_mixed) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t* __restrict__ sorted = srt.get();
  const uint32_t ix = sorted[p];
  const uint32_t b = n_tiles[ix] ? min((uint32_t)((keys[ix] - mm[0]) >> bs_shift(mm)), kBsInactive - 1u) : kBsInactive;
  if (b == kBsInactive || bmin[b] == ~bmax[b]) {  // inactive, or one key value: index order is the order
    order[p] = ix;
    return;
  }
  const uint32_t lo = start[b], hi = lo + count[b];
  if (hi - lo > (uint32_t)kBsRankBrute) {  // warp (<= kBsRankMax) or CTA sort
    if (p == lo) {
      if (hi - lo > (uint32_t)kBsRankMax) large[atomicAdd(n_large, 1u)] = b;
      else mixed[atomicAdd(n_mixed, 1u)] = b;
    }
    return;
  }
  const unsigned long long k = keys[ix];
  uint32_t r = 0;
  for (uint32_t q = lo; q < hi; ++q) {
    const uint32_t iq = sorted[q];
    r += bs_less(keys[iq], iq, k, ix);
  }
  order[lo + r] = ix;
}

// One CTA per large mixed bucket: bitonic sort by (key, index) with all
// comparators ascending (elements past the bucket's end - virtual +inf -
// never move and are skipped), in shared memory when it fits, else in
// place in global memory (scratch K / I).  Writes the bucket's order[].
__global__ void __launch_bounds__(kBsLargeThreads)
    k_bs_large(const unsigned long long* __restrict__ keys, BsSorted srt,
               const uint32_t* __restrict__ start, const uint32_t* __restrict__ count,
               const uint32_t* __restrict__ large,
               const uint32_t* __restrict__ n_large, unsigned long long* __restrict__ gk, uint32_t* __restrict__ gi,
               uint32_t* __restrict__ order) {
  extern __shared__ unsigned char bs_smem[];
  const uint32_t* __restrict__ sorted = srt.get();
  const uint32_t nl = *n_large;
  for (uint32_t j = blockIdx.x; j < nl; j += gridDim.x) {
    const uint32_t b = large[j];
    const uint32_t lo = start[b], s = count[b];
    uint32_t m = 1;
    while (m < s) m <<= 1;
    const bool in_smem = s <= (uint32_t)kBsSmemMax;
    unsigned long long* K = in_smem ? reinterpret_cast<unsigned long long*>(bs_smem) : gk + lo;
    uint32_t* I = in_smem ? reinterpret_cast<uint32_t*>(bs_smem + sizeof(unsigned long long) * kBsSmemMax) : gi + lo;
    for (uint32_t t = threadIdx.x; t < s; t += blockDim.x) {
      const uint32_t ix = sorted[lo + t];
      K[t] = keys[ix];
      I[t] = ix;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= m; k <<= 1) {
      for (uint32_t st = k >> 1; st > 0; st >>= 1) {
        const int ls = __ffs(st) - 1;
        for (uint32_t t = threadIdx.x; t < (m >> 1); t += blockDim.x) {
          const uint32_t blk = t >> ls, off = t & (st - 1);
          uint32_t a, c;
          if (st == (k >> 1)) {  // first step of a merge: mirrored pairs
            a = blk * k + off;
            c = blk * k + k - 1 - off;
          } else {
            a = (blk << (ls + 1)) + off;
            c = a + st;
          }
          if (c < s) {
            const unsigned long long ka = K[a], kc = K[c];
            const uint32_t ia = I[a], ic = I[c];
            if (bs_less(kc, ic, ka, ia)) {
              K[a] = kc;
              K[c] = ka;
              I[a] = ic;
              I[c] = ia;
            }
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t t = threadIdx.x; t < s; t += blockDim.x) order[lo + t] = I[t];
    __syncthreads();
  }
}

// One warp per mixed bucket of kBsRankBrute + 1 .. kBsRankMax splats: bitonic sort by
// (key, index) of kS * 32 register slots (element e = slot * 32 + lane;
// padding = +inf), cross-lane steps by shuffles, in-lane steps by swaps.
template <int kS>
__device__ __forceinline__ void bs_warp_sort(unsigned long long (&k)[kS], uint32_t (&ix)[kS]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32 * kS; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int sl = 0; sl < kS; ++sl) {
        const int e = sl * 32 + lane;
        const bool up = (e & size) == 0;  // ascending block
        if (j >= 32) {
          const int js = j >> 5;
          if ((sl & js) == 0) {  // pair (sl, sl ^ js) inside the lane, lower slot decides
            const int so = sl ^ js;
            const bool sw = up ? bs_less(k[so], ix[so], k[sl], ix[sl]) : bs_less(k[sl], ix[sl], k[so], ix[so]);
            if (sw) {
              const unsigned long long tk = k[sl];
              const uint32_t ti = ix[sl];
              k[sl] = k[so];
              ix[sl] = ix[so];
              k[so] = tk;
              ix[so] = ti;
            }
          }
        } else {
          const unsigned long long ok = __shfl_xor_sync(0xffffffffu, k[sl], j);
          const uint32_t oi = __shfl_xor_sync(0xffffffffu, ix[sl], j);
          const bool lower = (lane & j) == 0;
          const bool other_less = bs_less(ok, oi, k[sl], ix[sl]);
          // keep the min in the lower position of an ascending pair (max of a descending one)
          const bool take = (lower == up) ? other_less : !other_less && !(ok == k[sl] && oi == ix[sl]);
          if (take) {
            k[sl] = ok;
            ix[sl] = oi;
          }
        }
      }
    }
  }
}

template <int kS>
__device__ __forceinline__ void bs_warp_bucket(const unsigned long long* __restrict__ keys,
                                               const uint32_t* __restrict__ sorted, uint32_t lo, uint32_t s,
                                               uint32_t* __restrict__ order) {
  const int lane = threadIdx.x & 31;
  unsigned long long k[kS];
  uint32_t ix[kS];
#pragma unroll
  for (int sl = 0; sl < kS; ++sl) {
    const uint32_t e = sl * 32 + lane;
    ix[sl] = e < s ? sorted[lo + e] : 0xffffffffu;
    k[sl] = e < s ? keys[ix[sl]] : ~0ull;
  }
  bs_warp_sort<kS>(k, ix);
#pragma unroll
  for (int sl = 0; sl < kS; ++sl) {
    const uint32_t e = sl * 32 + lane;
    if (e < s) order[lo + e] = ix[sl];
  }
}

// A mixed bucket usually holds a few distinct depth values (exact ties of a
// lattice column each), every value's splats already in index order: the
// rank of a splat is (splats of smaller value) + (earlier splats of its
// value).  Two warp passes over the bucket in 32-splat chunks with a
// warp-uniform table of up to kBsDistinct values and their counts; more
// distinct values -> the register bitonic sort.
constexpr int kBsDistinct = 8;

__device__ __forceinline__ bool bs_warp_few(const unsigned long long* __restrict__ keys,
                                            const uint32_t* __restrict__ sorted, uint32_t lo, uint32_t s,
                                            uint32_t* __restrict__ order) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long val[kBsDistinct];
  uint32_t cnt[kBsDistinct], below[kBsDistinct];
  int nd = 0;
#pragma unroll
  for (int t = 0; t < kBsDistinct; ++t) {
    val[t] = 0;
    cnt[t] = 0;
  }
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      // below[t] = splats with a smaller value; cnt becomes the running count
#pragma unroll
      for (int t = 0; t < kBsDistinct; ++t) {
        uint32_t acc = 0;
#pragma unroll
        for (int u = 0; u < kBsDistinct; ++u) acc += (u < nd && val[u] < val[t]) ? cnt[u] : 0u;
        below[t] = acc;
      }
#pragma unroll
      for (int t = 0; t < kBsDistinct; ++t) cnt[t] = 0;
    }
    for (uint32_t c0 = 0; c0 < s; c0 += 32) {
      const bool valid = c0 + lane < s;
      const uint32_t ix = valid ? sorted[lo + c0 + lane] : 0u;
      const unsigned long long k = valid ? keys[ix] : 0ull;
      unsigned todo = __ballot_sync(0xffffffffu, valid);
      while (todo) {
        const int l = __ffs(todo) - 1;
        const unsigned long long kv = __shfl_sync(0xffffffffu, k, l);
        const unsigned grp = __ballot_sync(0xffffffffu, valid && k == kv);
        int slot = -1;
#pragma unroll
        for (int t = 0; t < kBsDistinct; ++t) slot = (t < nd && val[t] == kv) ? t : slot;
        if (slot < 0) {
          if (nd == kBsDistinct || pass == 1) return false;  // too many values (warp-uniform)
          slot = nd++;
#pragma unroll
          for (int t = 0; t < kBsDistinct; ++t) val[t] = t == slot ? kv : val[t];
        }
        uint32_t base = 0, bl = 0;
#pragma unroll
        for (int t = 0; t < kBsDistinct; ++t) {
          base = t == slot ? cnt[t] : base;
          bl = t == slot ? below[t] : bl;
          cnt[t] += t == slot ? (uint32_t)__popc(grp) : 0u;
        }
        if (pass == 1 && (grp >> lane) & 1u) order[lo + bl + base + __popc(grp & lt)] = ix;
        todo &= ~grp;
      }
    }
  }
  return true;
}

__global__ void __launch_bounds__(128) k_bs_mixed(const unsigned long long* __restrict__ keys, BsSorted srt,
                                                  const uint32_t* __restrict__ start,
                                                  const uint32_t* __restrict__ count,
                                                  const uint32_t* __restrict__ mixed,
                                                  const uint32_t* __restrict__ n_mixed,
                                                  uint32_t* __restrict__ order) {
  const uint32_t* __restrict__ sorted = srt.get();
  const uint32_t nm = *n_mixed;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < nm; j += warps) {
    const uint32_t b = mixed[j];
    const uint32_t lo = start[b], s = count[b];
    if (bs_warp_few(keys, sorted, lo, s, order)) continue;
    if (s <= 64) bs_warp_bucket<2>(keys, sorted, lo, s, order);
    else if (s <= 128) bs_warp_bucket<4>(keys, sorted, lo, s, order);
    else bs_warp_bucket<8>(keys, sorted, lo, s, order);
  }
}

}  // namespace

size_t bucket_sort_workspace_bytes(int64_t n) {
  return bs_fixed_bytes() + al256(scan_workspace_bytes(kBsBuckets)) + onesweep_workspace_bytes(n) + 256;
}

xg_status bucket_sort_depth(const unsigned long long* keys, const uint32_t* n_tiles, int64_t n,
                            unsigned long long* key_a, unsigned long long* key_b, uint32_t* val_a, uint32_t* val_b,
                            uint32_t* order, uint32_t* n_dev, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (n < 1) return XG_OK;
  BsWs w;
  if (!bs_carve(ws, ws_bytes, w) || w.tail_bytes < onesweep_workspace_bytes(n)) {
    set_error_msg("bucket_sort_depth: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  // two memsets: mm, bmin, bmax to all ones; the counts, the bucket-count
  // scan's look-back state and the onesweep's histograms / look-back state
  // to zero (bs_carve's layout)
  cudaMemsetAsync(w.mm, 0xff, (size_t)((char*)w.start - (char*)w.mm), s);
  cudaMemsetAsync(w.n_large, 0, (size_t)((char*)w.tail - (char*)w.n_large) + os_prepare_bytes(n, 2), s);
  const int g = (int)((n + 255) / 256);
  k_bs_minmax<<<g < 592 ? g : 592, 256, 0, s>>>(keys, n_tiles, n, w.mm, n_dev);
  xg_status st = check_launch("k_bs_minmax");
  if (st != XG_OK) return st;
  // bucket ids into key_b, iota into val_b (the onesweep's read-only inputs)
  // (the onesweep's histograms are accumulated by k_bs_bucket: zero them first)
  const OsWs ow = os_prepare(w.tail, n, 2, s, false);
  k_bs_bucket<<<g, 256, 0, s>>>(keys, n_tiles, n, w.mm, key_b, val_b, w.count, w.bmin, w.bmax, ow.ghist);
  if ((st = check_launch("k_bs_bucket")) != XG_OK) return st;

  // stable by 16-bit bucket id: two byte passes (ids < 2^16); no final copy
  k_os_scan<<<1, 256, 0, s>>>(ow.ghist, ow.gofs, n_dev, n, ow.sel, 2);
  if ((st = check_launch("k_os_scan")) != XG_OK) return st;
  if ((st = os_passes(ow, key_b, val_b, key_a, key_b, val_a, val_b, n, n_dev, 2, s)) != XG_OK) return st;
  BsSorted srt{{val_a, val_b, val_b}, ow.sel + kOsPasses};
#if XG_BS_BOUNDS
  k_bs_bounds<<<g, 256, 0, s>>>(keys, n_tiles, w.mm, srt, n, w.start);
  if ((st = check_launch("k_bs_bounds")) != XG_OK) return st;
#else
  g_scan_precleared = w.scan_bytes >= scan_workspace_bytes(kBsBuckets);  // (zeroed above)
  if ((st = scan_u32(w.count, nullptr, w.start, kBsBuckets, nullptr, kBsBuckets, nullptr, w.scan_ws, w.scan_bytes,
                     s)) != XG_OK)
    return st;
#endif
  k_bs_rank<<<g, 256, 0, s>>>(keys, n_tiles, w.mm, srt, n, w.start, w.count, w.bmin, w.bmax, order, w.large,
                              w.n_large, w.mixed, w.n_mixed);
  if ((st = check_launch("k_bs_rank")) != XG_OK) return st;
  k_bs_mixed<<<4 * 148, 128, 0, s>>>(keys, srt, w.start, w.count, w.mixed, w.n_mixed, order);
  if ((st = check_launch("k_bs_mixed")) != XG_OK) return st;
  static bool attr = false;
  const int smem = (int)((sizeof(unsigned long long) + sizeof(uint32_t)) * kBsSmemMax);
  if (!attr) {
    cudaFuncSetAttribute(k_bs_large, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  k_bs_large<<<148, kBsLargeThreads, smem, s>>>(keys, srt, w.start, w.count, w.large, w.n_large, key_a, val_a,
                                                 order);
  return check_launch("k_bs_large");
}

}  // namespace xg
