// Internal helpers shared by the libxgauss translation units (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/xgauss.h"

namespace xg {

constexpr int kTile = XG_TILE_SIZE;
constexpr double kLog2e = 1.4426950408889634073599246810019;
constexpr double kLn2 = 0.69314718055994530941723212145818;
// Power cut-off (-30) expressed on the log2 scale the kernels work in.
constexpr float kCut2 = (float)(XG_POWER_CUTOFF * kLog2e);
constexpr float kFloor = (float)XG_TRANSMITTANCE_FLOOR;
constexpr float kClamp = (float)XG_SIGMA_CLAMP;

// Remember the last error for xg_last_error().
void set_error(const char* what, cudaError_t err);
void set_error_msg(const char* what);
void note_launch();

// Called once after every kernel launch: error check + launch accounting
// (xg_kernel_launches(), used by bench.py's gpu_launches).
inline xg_status check_launch(const char* what) {
  note_launch();
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    set_error(what, err);
    return XG_ERR_CUDA;
  }
  return XG_OK;
}

// Heaviest-first tile schedule from the tile ranges (xg_composite.cu).
xg_status launch_tile_order(const int64_t* ranges, int n_tiles, int32_t* order, cudaStream_t s);

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

inline int tiles_x(const xg_camera& c) { return (c.width + kTile - 1) / kTile; }
inline int tiles_y(const xg_camera& c) { return (c.height + kTile - 1) / kTile; }

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------

// Hardware 2^x (MUFU.EX2, flush-to-zero).  The only approximate
// transcendental on the per-pair path; everything per-Gaussian is float64.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Vector reduction into global memory (sm_90+): one L2 atomic for 4 floats.
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

// Deterministic float64 exp shared by every per-Gaussian quantity (scales,
// sigmoids).  Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2, then a
// degree-13 Taylor polynomial in Horner form with fused multiply-adds:
// every step is an IEEE-754 correctly rounded operation, so host and
// device produce identical bits (libm exp and CUDA exp may not).
__host__ __device__ __forceinline__ double det_exp(double x) {
  if (!(x == x)) return x;            // NaN
  if (x > 709.0) return 1.0 / 0.0;    // overflow
  if (x < -745.0) return 0.0;         // underflow
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  double kd = (double)(long long)(x * 1.44269504088896338700e+00 + (x >= 0 ? 0.5 : -0.5));
  double r = fma(-kd, ln2_hi, x);
  r = fma(-kd, ln2_lo, r);
  // 1/n! coefficients
  double p = 1.6059043836821614599e-10;     // 1/13!
  p = fma(p, r, 2.0876756987868098979e-09);  // 1/12!
  p = fma(p, r, 2.5052108385441718775e-08);  // 1/11!
  p = fma(p, r, 2.7557319223985890653e-07);  // 1/10!
  p = fma(p, r, 2.7557319223985890653e-06);  // 1/9!
  p = fma(p, r, 2.4801587301587301587e-05);  // 1/8!
  p = fma(p, r, 1.9841269841269841270e-04);  // 1/7!
  p = fma(p, r, 1.3888888888888888889e-03);  // 1/6!
  p = fma(p, r, 8.3333333333333333333e-03);  // 1/5!
  p = fma(p, r, 4.1666666666666666667e-02);  // 1/4!
  p = fma(p, r, 1.6666666666666666667e-01);  // 1/3!
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  // scale by 2^k in two steps so subnormal results stay exact-rounded-ish
  long long k = (long long)kd;
  long long k1 = k / 2, k2 = k - k1;
  union { double d; unsigned long long u; } s1, s2;
  s1.u = (unsigned long long)(k1 + 1023) << 52;
  s2.u = (unsigned long long)(k2 + 1023) << 52;
  return (p * s1.d) * s2.d;
}

// Stable two-branch logistic (gaussians.py:29-38) on det_exp.
__host__ __device__ __forceinline__ double det_sigmoid(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + det_exp(-x));
  double e = det_exp(x);
  return e / (1.0 + e);
}

}  // namespace xg
