// The reference's kernel-backend contract at the reference's own precision:
// forward_tiles / backward_tiles of rasterizer/_kernels.pyx:23-178 on float64
// active-row arrays, with float64 arithmetic in the same operation order
// (compiled with -fmad=false: every product and sum rounds as the Cython
// loop's does on x86-64, which has no FMA contraction at -O3 without -march).
// The only differences from the compiled backend are the device exp() (<= 1
// ulp, libm's is correctly rounded in almost all cases) and, in the
// backward, the order in which the per-pixel terms of a splat are summed
// (warp shuffle tree + atomics instead of raster order): results agree with
// it to ~1e-15 relative, well inside the reference's own lockstep tolerance
// between its two backends (test_rasterizer.py:223-257: rtol 1e-12 forward,
// 1e-9 backward).
//
// These serve the plug-in point (xsplat's "cuda" backend, rasterizer/
// xsplat_backend.py); the engine's own render path composites in float32
// (xg_composite.cu).  One CTA per 16 x 16 tile, one thread per pixel, the
// tile's entries staged in shared memory 256 at a time, the CTA stopping
// once every pixel's transmittance is below the floor.
#include <math.h>

#include "xg_internal.cuh"

namespace xg {
namespace {

constexpr int kT = 16;
constexpr int kB = 256;  // entries staged per batch (one per thread)
constexpr double kCut = -30.0, kFloor64 = 1e-4, kClamp = 0.99;

struct Rec64 {
  double mx, my, a, b, c, i, o;
};

__device__ __forceinline__ void stage(Rec64* s, const double* __restrict__ m, const double* __restrict__ cn,
                                      const double* __restrict__ it, const double* __restrict__ op,
                                      const int32_t* __restrict__ entry, long long k, long long end, int* s_j) {
  if (k < end) {
    const int j = entry[k];
    s[threadIdx.x] = Rec64{m[2 * j], m[2 * j + 1], cn[3 * j], cn[3 * j + 1], cn[3 * j + 2], it[j], op[j]};
    s_j[threadIdx.x] = j;
  }
}

// _kernels.pyx:62-65 evaluated exactly as written
__device__ __forceinline__ double power_of(const Rec64& r, double fx, double fy, double& dx, double& dy) {
  dx = fx - r.mx;
  dy = fy - r.my;
  return -0.5 * (r.a * dx * dx + r.c * dy * dy) - r.b * dx * dy;
}

__global__ void __launch_bounds__(kB) k_forward_tiles64(int h, int w, const double* __restrict__ m,
                                                        const double* __restrict__ cn,
                                                        const double* __restrict__ it,
                                                        const double* __restrict__ op,
                                                        const int32_t* __restrict__ entry,
                                                        const long long* __restrict__ ranges,
                                                        double* __restrict__ image) {
  __shared__ Rec64 s[kB];
  __shared__ int s_j[kB];
  const int t = blockIdx.x, ntx = (w + kT - 1) / kT;
  const int px = (t % ntx) * kT + (threadIdx.x & 15), py = (t / ntx) * kT + (threadIdx.x >> 4);
  const bool in = px < w && py < h;
  const long long start = ranges[2 * t], end = ranges[2 * t + 1];
  const double fx = px, fy = py;
  double trans = 1.0, acc = 0.0;
  bool live = in;
  for (long long b0 = start; b0 < end; b0 += kB) {
    if (__syncthreads_or(live) == 0) break;
    stage(s, m, cn, it, op, entry, b0 + threadIdx.x, end, s_j);
    __syncthreads();
    const int cnt = (int)min((long long)kB, end - b0);
    for (int q = 0; q < cnt && live; ++q) {
      if (trans < kFloor64) {  // tested before every entry (_kernels.pyx:57-58)
        live = false;
        break;
      }
      const Rec64 r = s[q];
      double dx, dy;
      const double power = power_of(r, fx, fy, dx, dy);
      if (power > 0.0 || power < kCut) continue;
      double sigma = r.o * exp(power);
      if (sigma >= kClamp) sigma = kClamp;
      acc += r.i * sigma * trans;
      trans *= 1.0 - sigma;
    }
    __syncthreads();
  }
  if (in) image[(long long)py * w + px] = acc;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kB) k_backward_tiles64(int h, int w, const double* __restrict__ m,
                                                         const double* __restrict__ cn,
                                                         const double* __restrict__ it,
                                                         const double* __restrict__ op,
                                                         const int32_t* __restrict__ entry,
                                                         const long long* __restrict__ ranges,
                                                         const double* __restrict__ dl, double* __restrict__ g_mean,
                                                         double* __restrict__ g_conic, double* __restrict__ g_int,
                                                         double* __restrict__ g_alpha) {
  __shared__ Rec64 s[kB];
  __shared__ int s_j[kB];
  const int t = blockIdx.x, ntx = (w + kT - 1) / kT;
  const int lane = threadIdx.x & 31;
  const int px = (t % ntx) * kT + (threadIdx.x & 15), py = (t / ntx) * kT + (threadIdx.x >> 4);
  const bool in = px < w && py < h;
  const long long start = ranges[2 * t], end = ranges[2 * t + 1];
  const double fx = px, fy = py;
  const double g = in ? dl[(long long)py * w + px] : 0.0;
  // pass 1: replay the blend for the pixel's total (_kernels.pyx:121-140)
  double trans = 1.0, acc = 0.0;
  bool live = in;
  for (long long b0 = start; b0 < end; b0 += kB) {
    if (__syncthreads_or(live) == 0) break;
    stage(s, m, cn, it, op, entry, b0 + threadIdx.x, end, s_j);
    __syncthreads();
    const int cnt = (int)min((long long)kB, end - b0);
    for (int q = 0; q < cnt && live; ++q) {
      if (trans < kFloor64) {
        live = false;
        break;
      }
      const Rec64 r = s[q];
      double dx, dy;
      const double power = power_of(r, fx, fy, dx, dy);
      if (power > 0.0 || power < kCut) continue;
      double sigma = r.o * exp(power);
      if (sigma >= kClamp) sigma = kClamp;
      acc += r.i * sigma * trans;
      trans *= 1.0 - sigma;
    }
    __syncthreads();
  }
  // pass 2: front to back with the suffix formula (_kernels.pyx:142-177); the
  // warp visits every entry together, so each splat's 7 terms are summed
  // over the warp's pixels before one set of atomics
  trans = 1.0;
  double prefix = 0.0;
  live = in && g != 0.0;  // (a zero-upstream pixel adds exact zeros to every term)
  for (long long b0 = start; b0 < end; b0 += kB) {
    if (__syncthreads_or(live) == 0) break;
    stage(s, m, cn, it, op, entry, b0 + threadIdx.x, end, s_j);
    __syncthreads();
    const int cnt = (int)min((long long)kB, end - b0);
    for (int q = 0; q < cnt; ++q) {
      if (!__any_sync(0xffffffffu, live)) break;
      double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // g_int, g_alpha, g_mean x/y, g_conic 0/1/2
      bool hit = false;
      if (live) {
        if (trans < kFloor64) {
          live = false;
        } else {
          const Rec64 r = s[q];
          double dx, dy;
          const double power = power_of(r, fx, fy, dx, dy);
          if (!(power > 0.0 || power < kCut)) {
            const double dens = exp(power);
            double sigma = r.o * dens;
            const bool clamped = sigma >= kClamp;
            if (clamped) sigma = kClamp;
            const double weight = sigma * trans;
            const double contrib = r.i * weight;
            v[0] = g * weight;
            if (!clamped) {
              const double suffix = acc - prefix - contrib;
              const double d_sigma = g * (r.i * trans - suffix / (1.0 - sigma));
              v[1] = d_sigma * dens;
              const double g_power = d_sigma * r.o * dens;
              v[2] = g_power * (r.a * dx + r.b * dy);
              v[3] = g_power * (r.b * dx + r.c * dy);
              v[4] = -(0.5 * g_power * dx * dx);
              v[5] = -(g_power * dx * dy);
              v[6] = -(0.5 * g_power * dy * dy);
            }
            prefix += contrib;
            trans *= 1.0 - sigma;
            hit = true;
          }
        }
      }
      if (!__any_sync(0xffffffffu, hit)) continue;
#pragma unroll
      for (int i = 0; i < 7; ++i) v[i] = warp_sum(v[i]);
      if (lane == 0) {
        const int j = s_j[q];
        atomicAdd(g_int + j, v[0]);
        atomicAdd(g_alpha + j, v[1]);
        atomicAdd(g_mean + 2 * j, v[2]);
        atomicAdd(g_mean + 2 * j + 1, v[3]);
        atomicAdd(g_conic + 3 * j, v[4]);
        atomicAdd(g_conic + 3 * j + 1, v[5]);
        atomicAdd(g_conic + 3 * j + 2, v[6]);
      }
    }
    __syncthreads();
  }
}

xg_status check_tiles_args(int32_t h, int32_t w, const void* a, const void* b, const void* c, const void* d,
                           const void* e, const void* r, const void* out, const char* what) {
  if (h < 1 || w < 1 || !a || !b || !c || !d || !r || !out) {
    set_error_msg(what);
    return XG_ERR_INVALID;
  }
  (void)e;
  return XG_OK;
}

}  // namespace
}  // namespace xg

using namespace xg;

extern "C" {

xg_status xg_forward_tiles_f64(int32_t h, int32_t w, const double* means2d, const double* conics,
                               const double* intensities, const double* opacities, const int32_t* entry_splat,
                               int64_t n_entries, const int64_t* tile_ranges, int64_t n_splats, double* image,
                               void* stream) {
  xg_status st = check_tiles_args(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges, image,
                                  "xg_forward_tiles_f64: invalid argument");
  if (st != XG_OK) return st;
  const int n_tiles = ((w + kT - 1) / kT) * ((h + kT - 1) / kT);
  cudaMemsetAsync(image, 0, sizeof(double) * (size_t)h * (size_t)w, (cudaStream_t)stream);
  if (n_entries < 1 || n_splats < 1) return XG_OK;
  k_forward_tiles64<<<n_tiles, kB, 0, (cudaStream_t)stream>>>(h, w, means2d, conics, intensities, opacities,
                                                              entry_splat, (const long long*)tile_ranges, image);
  return check_launch("k_forward_tiles64");
}

xg_status xg_backward_tiles_f64(int32_t h, int32_t w, const double* means2d, const double* conics,
                                const double* intensities, const double* opacities, const int32_t* entry_splat,
                                int64_t n_entries, const int64_t* tile_ranges, int64_t n_splats,
                                const double* dl_dimage, double* g_mean, double* g_conic, double* g_int,
                                double* g_alpha, void* stream) {
  xg_status st = check_tiles_args(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges,
                                  dl_dimage, "xg_backward_tiles_f64: invalid argument");
  if (st != XG_OK) return st;
  if (!g_mean || !g_conic || !g_int || !g_alpha) {
    set_error_msg("xg_backward_tiles_f64: invalid argument");
    return XG_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t n = n_splats > 0 ? (size_t)n_splats : 0;
  cudaMemsetAsync(g_mean, 0, sizeof(double) * 2 * n, s);
  cudaMemsetAsync(g_conic, 0, sizeof(double) * 3 * n, s);
  cudaMemsetAsync(g_int, 0, sizeof(double) * n, s);
  cudaMemsetAsync(g_alpha, 0, sizeof(double) * n, s);
  if (n_entries < 1 || n_splats < 1) return XG_OK;
  const int n_tiles = ((w + kT - 1) / kT) * ((h + kT - 1) / kT);
  k_backward_tiles64<<<n_tiles, kB, 0, s>>>(h, w, means2d, conics, intensities, opacities, entry_splat,
                                            (const long long*)tile_ranges, dl_dimage, g_mean, g_conic, g_int,
                                            g_alpha);
  return check_launch("k_backward_tiles64");
}

}  // extern "C"
