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

size_t scan_workspace_bytes(int64_t cap) {
  const int64_t tiles = (cap + kScanTile - 1) / kScanTile + 1;
  return align_up(sizeof(unsigned long long) * (size_t)tiles) + 256;
}

xg_status scan_u32(const uint32_t* in, const uint32_t* gather, uint32_t* out, int64_t cap,
                   const uint32_t* n_dev, int64_t n_host, uint32_t* total, void* ws, size_t ws_bytes,
                   cudaStream_t s) {
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
  cudaMemsetAsync(ws, 0, need, s);
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
              uint32_t* __restrict__ ghist) {
  __shared__ uint32_t h[kOsPasses][256];
  for (int i = threadIdx.x; i < kOsPasses * 256; i += kOsThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  long long n = *n_dev;
  if (n > cap) n = cap;
  for (long long i = (long long)blockIdx.x * kOsThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kOsThreads) {
    const unsigned long long k = keys[i];
#pragma unroll
    for (int p = 0; p < kOsPasses; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
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
                                                 const uint32_t* n_dev, long long cap, int* __restrict__ sel) {
  __shared__ uint32_t s[256];
  __shared__ int trivial[kOsPasses];
  long long n = *n_dev;
  if (n > cap) n = cap;
  const int d = threadIdx.x;
  for (int p = 0; p < kOsPasses; ++p) {
    const uint32_t v = ghist[p * 256 + d];
    const int t = __syncthreads_or((long long)v == n);
    if (d == 0) trivial[p] = t;
    s[d] = v;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {  // inclusive Hillis-Steele
      const uint32_t x = d >= o ? s[d - o] : 0u;
      __syncthreads();
      s[d] += x;
      __syncthreads();
    }
    gofs[p * 256 + d] = s[d] - v;
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
  const unsigned long long* kin = a.keys[src];
  const uint32_t* vin = a.vals[src];
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
  unsigned long long* kout = a.keys[a.sel[p + 1]];
  uint32_t* vout = a.vals[a.sel[p + 1]];
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
                            const uint32_t* n_dev, long long cap, const int* sel) {
  const int r = sel[kOsPasses];
  const uint32_t* src = r == 0 ? vals_a : r == 1 ? vals_b : nullptr;
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

xg_status onesweep_sort_pairs64(const unsigned long long* keys_in, const uint32_t* vals_in,
                                unsigned long long* keys_a, unsigned long long* keys_b, uint32_t* vals_a,
                                uint32_t* vals_b, uint32_t* vals_out, int64_t cap, const uint32_t* n_dev,
                                void* ws, size_t ws_bytes, cudaStream_t s) {
  if (cap <= 0) return XG_OK;
  if (ws_bytes < onesweep_workspace_bytes(cap)) {
    set_error_msg("onesweep_sort_pairs64: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  const int64_t tiles = (cap + kOsTile - 1) / kOsTile;
  char* p = (char*)ws;
  uint32_t* ghist = (uint32_t*)p;
  uint32_t* gofs = ghist + kOsPasses * 256;
  p += align_up(sizeof(uint32_t) * kOsPasses * 256 * 2);
  int* sel = (int*)p;
  p += align_up(sizeof(int) * (kOsPasses + 1));
  uint32_t* ctr = (uint32_t*)p;
  p += align_up(sizeof(uint32_t) * kOsPasses);
  uint32_t* status = (uint32_t*)p;
  cudaMemsetAsync(ws, 0, onesweep_workspace_bytes(cap), s);
  const int hgrid = (int)(tiles < 296 ? tiles : 296);
  k_os_hist<<<hgrid, kOsThreads, 0, s>>>(keys_in, n_dev, cap, ghist);
  xg_status st = check_launch("k_os_hist");
  if (st != XG_OK) return st;
  k_os_scan<<<1, 256, 0, s>>>(ghist, gofs, n_dev, cap, sel);
  if ((st = check_launch("k_os_scan")) != XG_OK) return st;
  for (int pass = 0; pass < kOsPasses; ++pass) {
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
    a.ghist = ghist;
    a.gofs = gofs;
    a.sel = sel;
    a.status = status + (size_t)pass * tiles * 256;
    a.tile_ctr = ctr + pass;
    k_os_pass<<<(int)tiles, kOsThreads, 0, s>>>(a);
    if ((st = check_launch("k_os_pass")) != XG_OK) return st;
  }
  k_os_finish<<<(int)(tiles < 296 ? tiles : 296), 256, 0, s>>>(vals_out, vals_a, vals_b, n_dev, cap, sel);
  return check_launch("k_os_finish");
}

}  // namespace xg
