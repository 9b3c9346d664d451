// K5: the data-parallel gradient exchange fused with Adam, over peer memory.
//
// One process per GPU; every rank's flat gradient, exchange buffer and sync
// words are mapped into every process (CUDA IPC, parallel.PeerExchange).  A
// data-parallel step (the summed per-view gradients, then Adam
// on identical replicas) is two kernels instead of a bucketed NCCL
// all-reduce followed by the Adam launches:
//
//   k_peer_reduce_scatter  signal "gradient ready" to every rank, wait for
//                          all signals, sum slice `rank` of the flat buffer
//                          over the ranks in rank order (peer loads) into the
//                          exchange buffer, OR the slice's per-field
//                          non-finite bits into every rank's status word,
//                          signal "arrived";
//   k_peer_allgather_adam  wait for every "arrived", read each slice of the
//                          summed gradient from its owner (peer loads) and
//                          apply the fused Adam of xg_adam_range to the whole
//                          buffer with the global non-finite bits.
//
// The exchange is two-shot (reduce-scatter, all-gather) like a ring
// all-reduce in bytes moved per rank, with the optimizer as the all-gather's
// epilogue: the gradient never round-trips through a separate all-reduce
// output.  Every rank adds the same values in the same order, so replicas
// stay bit-identical.  Epoch protocol (epoch = 1, 2, ... per exchange, the
// counters only grow): "ready" and "arrived" are per-rank counters that
// every rank increments once per epoch; a rank proceeds when its counter
// reaches world * epoch.  The exchange slot and status word alternate by
// epoch parity; a rank clears the previous parity's status word before it
// signals ready - no peer can write that word again until this rank's next
// ready signal.  Waits are bounded: after ~10 s a kernel sets
// XG_ST_PEER_TIMEOUT in the caller's sticky word and returns (no hang).
#include "xg_internal.cuh"

namespace xg {
namespace {

constexpr int kSyncReady = 0, kSyncArrived = 1, kSyncStatus = 2, kSyncCtaDone = 4, kSyncBad = 5;
constexpr long long kSpinCycles = 20000000000ll;  // ~10 s at 1.9 GHz

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// thread 0 of each CTA waits until *ctr >= target; false on timeout
__device__ __forceinline__ bool wait_count(const uint32_t* ctr, uint32_t target, uint32_t* sticky) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    int ok = 1;
    while ((int)(ld_acquire_sys(ctr) - target) < 0) {
      if (clock64() - t0 > kSpinCycles) {
        ok = 0;
        atomicOr(sticky, XG_ST_PEER_TIMEOUT);
        break;
      }
      __nanosleep(256);
    }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

struct PeerArgs {
  xg_peer_group pg;
  long long total, slice;  // flat elements, slice length (multiple of 4)
  long long bounds[4];     // 3n, 7n, 10n, 11n
  uint32_t* sticky;
};

__device__ __forceinline__ int field_of(const long long (&b)[4], long long e) {
  return (e >= b[0]) + (e >= b[1]) + (e >= b[2]) + (e >= b[3]);
}

__global__ void __launch_bounds__(256) k_peer_reduce_scatter(PeerArgs a) {
  const int rank = a.pg.rank, world = a.pg.world;
  const uint32_t epoch = a.pg.epoch, par = epoch & 1u;
  uint32_t* const me = a.pg.sync[rank];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    me[kSyncStatus + (par ^ 1u)] = 0u;  // the previous epoch's status word (see the protocol above)
    __threadfence_system();
    for (int k = 0; k < world; ++k) atomicAdd_system(a.pg.sync[k] + kSyncReady, 1u);
  }
  if (!wait_count(me + kSyncReady, (uint32_t)world * epoch, a.sticky)) return;
  const long long lo = (long long)rank * a.slice, hi = min(lo + a.slice, a.total);
  float* const out = a.pg.xbuf[rank] + (long long)par * a.slice;
  unsigned bad = 0;
  for (long long e = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; e < hi;
       e += (long long)gridDim.x * blockDim.x) {
    float s = a.pg.grads[0][e];
    for (int k = 1; k < world; ++k) s += a.pg.grads[k][e];  // rank order on every rank
    out[e - lo] = s;
    if (!isfinite(s)) bad |= 1u << field_of(a.bounds, e);
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && (threadIdx.x & 31) == 0) atomicOr(me + kSyncBad, bad);
  // the last CTA publishes the slice's bits to every rank and signals arrival
  __threadfence_system();  // (this CTA's slice sums, before its done count)
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t done = atomicAdd(me + kSyncCtaDone, 1u) + 1u;
    if (done % gridDim.x == 0u) {
      __threadfence();
      const uint32_t slice_bad = atomicExch(me + kSyncBad, 0u);
      if (slice_bad)
        for (int k = 0; k < world; ++k) atomicOr_system(a.pg.sync[k] + kSyncStatus + par, slice_bad);
      __threadfence_system();
      for (int k = 0; k < world; ++k) atomicAdd_system(a.pg.sync[k] + kSyncArrived, 1u);
    }
  }
}

struct AdamPeerArgs {
  PeerArgs p;
  float* param;
  float* m;
  float* v;
  float lr[5];
  float b1, b2, omb1, omb2, bc1, bc2, eps;
};

__global__ void __launch_bounds__(256) k_peer_allgather_adam(AdamPeerArgs a) {
  const xg_peer_group& pg = a.p.pg;
  const uint32_t epoch = pg.epoch, par = epoch & 1u;
  uint32_t* const me = pg.sync[pg.rank];
  const uint32_t before = *a.p.sticky;  // (bits of earlier steps: the trainer raises on them)
  if (!wait_count(me + kSyncArrived, (uint32_t)pg.world * epoch, a.p.sticky)) return;
  const uint32_t bad = ld_acquire_sys(me + kSyncStatus + par) | ((before >> XG_ST_GRAD_NONFINITE_SHIFT) & 0x1fu);
  if (blockIdx.x == 0 && threadIdx.x == 0 && bad) atomicOr(a.p.sticky, bad << XG_ST_GRAD_NONFINITE_SHIFT);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < a.p.total;
       e += (long long)gridDim.x * blockDim.x) {
    const int f = field_of(a.p.bounds, e);
    if (bad & ((2u << f) - 1u)) continue;  // a field <= f diverged (trainer.py:158-170)
    const int owner = (int)(e / a.p.slice);
    const float g = pg.xbuf[owner][(long long)par * a.p.slice + (e - (long long)owner * a.p.slice)];
    // (the arithmetic of k_adam, xg_optim.cu)
    float m = a.m[e], v = a.v[e];
    m = __fmaf_rn(a.b1, m, __fmul_rn(a.omb1, g));
    v = __fmaf_rn(a.b2, v, __fmul_rn(__fmul_rn(a.omb2, g), g));
    a.m[e] = m;
    a.v[e] = v;
    a.param[e] = __fsub_rn(
        a.param[e], __fmul_rn(a.lr[f], __fdiv_rn(__fdiv_rn(m, a.bc1), __fadd_rn(__fsqrt_rn(__fdiv_rn(v, a.bc2)), a.eps))));
  }
}

bool make_peer_args(const xg_peer_group* pg, int64_t n, int32_t nf, uint32_t* sticky, PeerArgs& a) {
  if (!pg || !sticky || n < 1 || nf < 1 || pg->world < 1 || pg->world > XG_PEER_MAX || pg->rank < 0 ||
      pg->rank >= pg->world || pg->epoch == 0)
    return false;
  for (int k = 0; k < pg->world; ++k)
    if (!pg->grads[k] || !pg->xbuf[k] || !pg->sync[k]) return false;
  a.pg = *pg;
  a.total = n * (11 + (int64_t)nf);
  a.slice = xg_peer_slice(n, nf, pg->world);
  a.bounds[0] = 3 * n;
  a.bounds[1] = 7 * n;
  a.bounds[2] = 10 * n;
  a.bounds[3] = 11 * n;
  a.sticky = sticky;
  return true;
}

int peer_grid(long long work) {
  const long long g = (work + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}

}  // namespace
}  // namespace xg

using namespace xg;

extern "C" {

int64_t xg_peer_slice(int64_t n, int32_t n_features, int32_t world) {
  if (n < 1 || n_features < 1 || world < 1) return 0;
  const int64_t total = n * (11 + (int64_t)n_features);
  return (((total + world - 1) / world) + 3) & ~(int64_t)3;
}

xg_status xg_peer_reduce_scatter(const xg_peer_group* pg, int64_t n, int32_t n_features, uint32_t* sticky,
                                 void* stream) {
  PeerArgs a;
  if (!make_peer_args(pg, n, n_features, sticky, a)) {
    set_error_msg("xg_peer_reduce_scatter: invalid argument");
    return XG_ERR_INVALID;
  }
  k_peer_reduce_scatter<<<peer_grid(a.slice), 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch("k_peer_reduce_scatter");
}

xg_status xg_peer_allgather_adam(const xg_peer_group* pg, float* params, float* exp_avg, float* exp_avg_sq,
                                 int64_t n, int32_t n_features, const double* lr, double beta1, double beta2,
                                 double eps, double bc1, double bc2, uint32_t* sticky, void* stream) {
  AdamPeerArgs a;
  if (!make_peer_args(pg, n, n_features, sticky, a.p) || !params || !exp_avg || !exp_avg_sq || !lr) {
    set_error_msg("xg_peer_allgather_adam: invalid argument");
    return XG_ERR_INVALID;
  }
  a.param = params;
  a.m = exp_avg;
  a.v = exp_avg_sq;
  for (int f = 0; f < 5; ++f) a.lr[f] = (float)lr[f];
  a.b1 = (float)beta1;
  a.b2 = (float)beta2;
  a.omb1 = (float)(1.0 - beta1);
  a.omb2 = (float)(1.0 - beta2);
  a.bc1 = (float)bc1;
  a.bc2 = (float)bc2;
  a.eps = (float)eps;
  k_peer_allgather_adam<<<peer_grid(a.p.total), 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch("k_peer_allgather_adam");
}

}  // extern "C"
