// SSIM loss and its exact pixel gradient (the training loss for gamma > 0).
//
// Reference semantics (pkg/src/xsplat/metrics.py:57-124, trainer.py:109-123):
//   mu_x = x (*) w, mu_y = y (*) w, var_x = x^2 (*) w - mu_x^2,
//   var_y = y^2 (*) w - mu_y^2, cov = xy (*) w - mu_x mu_y   ('valid' windows,
//   w = 11x11 Gaussian, sigma 1.5, normalised), c1 = (0.01 R)^2, c2 = (0.03 R)^2,
//   s = (2 mu_x mu_y + c1)(2 cov + c2) / ((mu_x^2 + mu_y^2 + c1)(var_x + var_y + c2)),
//   SSIM = mean(s); dSSIM/dx = full-convolutions of the per-window partials
//   g_mu, g_q, g_r with w, combined as G_mu + 2 x G_q + y G_r.
//
// B200 mapping.  Three small kernels, all float64 arithmetic (the reference
// is float64; B200's FP64 pipe makes the 11-tap separable filters free at
// detector sizes), inputs float32 or float64:
//   S1  per 32x32 tile of window positions: stage a 42x42 input patch in
//       shared memory, horizontal 11-tap pass of the five moments (x, y,
//       x^2, y^2, xy) into shared memory, vertical pass -> s and the three
//       partial maps (to the workspace) and a per-CTA partial sum of s
//   S2  per 32x32 tile of pixels: the three partial maps' 42x42
//       neighbourhood (zero outside the valid range) through the same
//       separable filter -> gradient, written as float64 and / or fused
//       into the trainer's float32 upstream gradient
//       dl = ssim_scale * dSSIM/dx + l1_scale * sign(x - y)
//   S3  deterministic in-order sum of the per-CTA partials -> mean SSIM
#include "xg_internal.cuh"

namespace xg {
namespace {

constexpr int kWin = 11;
constexpr int kHalo = kWin - 1;
constexpr int kST = 32;              // tile edge (outputs)
constexpr int kSP = kST + kHalo;     // staged patch edge
constexpr int kSThreads = 256;

struct SsimW {
  double g[kWin];
};

// Normalised 1-D factors of the separable window (gaussian_window,
// metrics.py:47-54: outer(g, g) / sum = (g / sum g) (g / sum g)^T).
SsimW window_1d() {
  SsimW w;
  double s = 0.0;
  for (int i = 0; i < kWin; ++i) {
    const double c = i - 0.5 * (kWin - 1);
    w.g[i] = exp(-(c * c) / (2.0 * 1.5 * 1.5));
    s += w.g[i];
  }
  for (int i = 0; i < kWin; ++i) w.g[i] /= s;
  return w;
}

template <typename T>
__global__ void __launch_bounds__(kSThreads) k_ssim_stats(const T* __restrict__ x, const T* __restrict__ y, int h,
                                                          int w, double c1, double c2, SsimW wg,
                                                          double* __restrict__ gmu, double* __restrict__ gq,
                                                          double* __restrict__ gr, double* __restrict__ partial,
                                                          double inv_count) {
  extern __shared__ double sm[];
  double* px = sm;                       // [kSP][kSP]
  double* py = px + kSP * kSP;           // [kSP][kSP]
  double* hs = py + kSP * kSP;           // [5][kSP][kST]
  __shared__ double red[kSThreads / 32];
  const int hv = h - kHalo, wv = w - kHalo;  // valid window positions
  const int r0 = blockIdx.y * kST, c0 = blockIdx.x * kST;
  for (int i = threadIdx.x; i < kSP * kSP; i += kSThreads) {
    const int r = r0 + i / kSP, c = c0 + i % kSP;
    const bool in = r < h && c < w;
    px[i] = in ? (double)x[(long long)r * w + c] : 0.0;
    py[i] = in ? (double)y[(long long)r * w + c] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSP * kST; i += kSThreads) {
    const int r = i / kST, c = i % kST;
    double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const double a = px[r * kSP + c + k], b = py[r * kSP + c + k], g = wg.g[k];
      m0 = fma(g, a, m0);
      m1 = fma(g, b, m1);
      m2 = fma(g, a * a, m2);
      m3 = fma(g, b * b, m3);
      m4 = fma(g, a * b, m4);
    }
    hs[0 * kSP * kST + i] = m0;
    hs[1 * kSP * kST + i] = m1;
    hs[2 * kSP * kST + i] = m2;
    hs[3 * kSP * kST + i] = m3;
    hs[4 * kSP * kST + i] = m4;
  }
  __syncthreads();
  double acc = 0.0;
  for (int i = threadIdx.x; i < kST * kST; i += kSThreads) {
    const int r = i / kST, c = i % kST;
    const int gr_ = r0 + r, gc = c0 + c;
    if (gr_ >= hv || gc >= wv) continue;
    double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const double g = wg.g[k];
#pragma unroll
      for (int q = 0; q < 5; ++q) m[q] = fma(g, hs[q * kSP * kST + (r + k) * kST + c], m[q]);
    }
    const double mx = m[0], my = m[1];
    const double vx = m[2] - mx * mx, vy = m[3] - my * my, cv = m[4] - mx * my;
    const double a1 = 2.0 * mx * my + c1, a2 = 2.0 * cv + c2;
    const double b1 = mx * mx + my * my + c1, b2 = vx + vy + c2;
    const double den = b1 * b2;
    const double s = a1 * a2 / den;
    acc += s;
    if (gmu) {
      const long long o = (long long)gr_ * wv + gc;
      gmu[o] = inv_count * (2.0 * my * (a2 - a1) / den + 2.0 * mx * s * (1.0 / b2 - 1.0 / b1));
      gq[o] = -inv_count * s / b2;
      gr[o] = 2.0 * inv_count * a1 / den;
    }
  }
  // deterministic block sum
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kSThreads / 32; ++k) t += red[k];
    partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

template <typename T>
__global__ void __launch_bounds__(kSThreads) k_ssim_grad(const T* __restrict__ x, const T* __restrict__ y, int h,
                                                         int w, SsimW wg, const double* __restrict__ gmu,
                                                         const double* __restrict__ gq,
                                                         const double* __restrict__ gr, double* __restrict__ grad,
                                                         float* __restrict__ dl, double ssim_scale,
                                                         double l1_scale) {
  extern __shared__ double sm[];
  double* pm = sm;                     // [3][kSP][kSP]
  double* hs = pm + 3 * kSP * kSP;     // [3][kSP][kST]
  const int hv = h - kHalo, wv = w - kHalo;
  const int r0 = blockIdx.y * kST, c0 = blockIdx.x * kST;
  // pixel p receives window q = p - k for k in [0, 10]^2: stage maps over
  // [r0 - 10, r0 + 31] x [c0 - 10, c0 + 31]
  for (int i = threadIdx.x; i < kSP * kSP; i += kSThreads) {
    const int r = r0 - kHalo + i / kSP, c = c0 - kHalo + i % kSP;
    const bool in = r >= 0 && c >= 0 && r < hv && c < wv;
    const long long o = (long long)r * wv + c;
    pm[i] = in ? gmu[o] : 0.0;
    pm[kSP * kSP + i] = in ? gq[o] : 0.0;
    pm[2 * kSP * kSP + i] = in ? gr[o] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSP * kST; i += kSThreads) {
    const int r = i / kST, c = i % kST;
    double m0 = 0.0, m1 = 0.0, m2 = 0.0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const double g = wg.g[kHalo - k];  // convolution (the window is symmetric)
      m0 = fma(g, pm[r * kSP + c + k], m0);
      m1 = fma(g, pm[kSP * kSP + r * kSP + c + k], m1);
      m2 = fma(g, pm[2 * kSP * kSP + r * kSP + c + k], m2);
    }
    hs[i] = m0;
    hs[kSP * kST + i] = m1;
    hs[2 * kSP * kST + i] = m2;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kST * kST; i += kSThreads) {
    const int r = i / kST, c = i % kST;
    const int pr = r0 + r, pc = c0 + c;
    if (pr >= h || pc >= w) continue;
    double m0 = 0.0, m1 = 0.0, m2 = 0.0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
      const double g = wg.g[kHalo - k];
      m0 = fma(g, hs[(r + k) * kST + c], m0);
      m1 = fma(g, hs[kSP * kST + (r + k) * kST + c], m1);
      m2 = fma(g, hs[2 * kSP * kST + (r + k) * kST + c], m2);
    }
    const long long o = (long long)pr * w + pc;
    const double xv = (double)x[o], yv = (double)y[o];
    const double gv = m0 + 2.0 * xv * m1 + yv * m2;
    if (grad) grad[o] = gv;
    if (dl) dl[o] = (float)(ssim_scale * gv + l1_scale * (double)((xv > yv) - (xv < yv)));
  }
}

__global__ void k_ssim_finish(const double* __restrict__ partial, int n, double inv_count, double* out) {
  __shared__ double red[32];
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += partial[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    *out = s * inv_count;
  }
}

size_t al8(size_t x) { return (x + 255) & ~(size_t)255; }

size_t ws_layout(int32_t h, int32_t w, size_t* off_maps, size_t* off_part) {
  const size_t hv = (size_t)(h - kHalo), wv = (size_t)(w - kHalo);
  const size_t tiles = ((wv + kST - 1) / kST) * ((hv + kST - 1) / kST);
  const size_t maps = al8(3 * sizeof(double) * hv * wv);
  if (off_maps) *off_maps = 0;
  if (off_part) *off_part = maps;
  return maps + al8(sizeof(double) * tiles) + 256;
}

template <typename T>
xg_status ssim_impl(const T* x, const T* y, int32_t h, int32_t w, double data_range, double* ssim_out,
                    double* grad, float* dl, double ssim_scale, double l1_scale, void* ws, size_t ws_bytes,
                    cudaStream_t s) {
  size_t om, op;
  const size_t need = ws_layout(h, w, &om, &op);
  if (ws_bytes < need) {
    set_error_msg("xg_ssim: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  const int hv = h - kHalo, wv = w - kHalo;
  const double c1 = (0.01 * data_range) * (0.01 * data_range), c2 = (0.03 * data_range) * (0.03 * data_range);
  const double inv = 1.0 / ((double)hv * (double)wv);
  double* maps = (double*)((char*)ws + om);
  double* gmu = maps;
  double* gq = gmu + (size_t)hv * wv;
  double* gr = gq + (size_t)hv * wv;
  double* part = (double*)((char*)ws + op);
  const bool want_grad = grad || dl;
  const SsimW wg = window_1d();
  const dim3 g1((wv + kST - 1) / kST, (hv + kST - 1) / kST);
  const size_t sm1 = sizeof(double) * (2 * kSP * kSP + 5 * kSP * kST);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ssim_stats<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    cudaFuncSetAttribute(k_ssim_stats<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    const int sm2 = (int)(sizeof(double) * (3 * kSP * kSP + 3 * kSP * kST));
    cudaFuncSetAttribute(k_ssim_grad<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    cudaFuncSetAttribute(k_ssim_grad<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    attr = true;
  }
  k_ssim_stats<T><<<g1, kSThreads, sm1, s>>>(x, y, h, w, c1, c2, wg, want_grad ? gmu : nullptr, gq, gr, part, inv);
  xg_status st = check_launch("k_ssim_stats");
  if (st != XG_OK) return st;
  if (ssim_out) {
    k_ssim_finish<<<1, 256, 0, s>>>(part, (int)(g1.x * g1.y), inv, ssim_out);
    if ((st = check_launch("k_ssim_finish")) != XG_OK) return st;
  }
  if (!want_grad) return XG_OK;
  const dim3 g2((w + kST - 1) / kST, (h + kST - 1) / kST);
  const size_t sm2 = sizeof(double) * (3 * kSP * kSP + 3 * kSP * kST);
  k_ssim_grad<T><<<g2, kSThreads, sm2, s>>>(x, y, h, w, wg, gmu, gq, gr, grad, dl, ssim_scale, l1_scale);
  return check_launch("k_ssim_grad");
}

}  // namespace
}  // namespace xg

using namespace xg;

extern "C" {

size_t xg_ssim_workspace_bytes(int32_t h, int32_t w) {
  if (h < kWin || w < kWin) return 256;
  return ws_layout(h, w, nullptr, nullptr);
}

xg_status xg_ssim(const void* pred, const void* ref, int32_t is_f64, int32_t h, int32_t w, double data_range,
                  double* ssim_out, double* grad_out, float* dl_out, double dl_ssim_scale, double dl_l1_scale,
                  void* workspace, size_t workspace_bytes, void* stream) {
  if (!pred || !ref || !workspace || h < kWin || w < kWin || !(data_range > 0.0)) {
    set_error_msg("xg_ssim: invalid argument (images must be at least 11 x 11)");
    return XG_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (is_f64)
    return ssim_impl((const double*)pred, (const double*)ref, h, w, data_range, ssim_out, grad_out, dl_out,
                     dl_ssim_scale, dl_l1_scale, workspace, workspace_bytes, s);
  return ssim_impl((const float*)pred, (const float*)ref, h, w, data_range, ssim_out, grad_out, dl_out,
                   dl_ssim_scale, dl_l1_scale, workspace, workspace_bytes, s);
}

}  // extern "C"
