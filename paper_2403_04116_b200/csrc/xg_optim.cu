// K4c fused Adam and K4d density control (trainer.py:147-268).
//
// Adam: one thread per Gaussian walks its 11 + N_f parameters (all fields
// live in one flat buffer, so the per-field rows are contiguous and a warp
// touches contiguous cache lines), updates moments and parameters, and
// renormalises the quaternion in the same pass - one read of p, m, v, g
// and one write of p, m, v per element, the HBM minimum (28 B/element).
// Arithmetic is float32 with IEEE division / square root (the moments are
// stored in float32; the update differs from the reference's float64 by a
// few ulp of the lr-scaled step).
//
// Density control: a mark kernel evaluates the clone / split / prune masks
// (float64 comparisons, so identical to the reference on the same inputs)
// and counts them; the host then applies the cap rule and calls apply,
// which scans the three masks and scatters keep / clone / split-child rows
// into the new [keep | clone | split x2] layout.
#include <math.h>
#include <stdint.h>

#include "xg_sort.cuh"

namespace xg {
namespace {

constexpr int kFields = 5;

struct Layout {
  long long off[kFields];
  int width[kFields];
};

__host__ Layout make_layout(long long n, int nf) {
  Layout L;
  const int w[kFields] = {3, 4, 3, 1, nf};
  long long o = 0;
  for (int f = 0; f < kFields; ++f) {
    L.off[f] = o;
    L.width[f] = w[f];
    o += n * w[f];
  }
  return L;
}

struct AdamArgs {
  float* p;
  const float* g;
  float* m;
  float* v;
  long long n;
  long long bound[4];  // field boundaries 3n, 7n, 10n, 11n of the flat layout
  long long begin, end;
  double lr[kFields];
  double b1, b2, eps, bc1, bc2;
  const uint32_t* status;
};

// Element-wise over [begin, end) of the flat buffer: coalesced, one read of
// p, m, v, g and one write of p, m, v per element (28 B, the HBM minimum).
// A range form lets data-parallel training run Adam on one gradient bucket
// while the next bucket is still being all-reduced.
__global__ void k_adam(AdamArgs a) {
  const uint32_t bad = a.status ? (a.status[0] >> XG_ST_GRAD_NONFINITE_SHIFT) & 0x1f : 0u;
  const float b1 = (float)a.b1, b2 = (float)a.b2, omb1 = (float)(1.0 - a.b1), omb2 = (float)(1.0 - a.b2);
  const float bc1 = (float)a.bc1, bc2 = (float)a.bc2, eps = (float)a.eps;
  float lrf[kFields];
#pragma unroll
  for (int k = 0; k < kFields; ++k) lrf[k] = (float)a.lr[k];
  for (long long e = a.begin + (long long)blockIdx.x * blockDim.x + threadIdx.x; e < a.end;
       e += (long long)gridDim.x * blockDim.x) {
    const int f = (e >= a.bound[0]) + (e >= a.bound[1]) + (e >= a.bound[2]) + (e >= a.bound[3]);
    if (bad & ((2u << f) - 1u)) continue;  // a field <= f diverged (the reference raises there)
    // float32 arithmetic (IEEE division and square root): the moments are
    // stored in float32 anyway, and the update differs from the reference's
    // float64 evaluation by a few ulp of the (lr-scaled) step only
    const float g = a.g[e];
    float m = a.m[e], v = a.v[e];
    m = __fmaf_rn(b1, m, __fmul_rn(omb1, g));
    v = __fmaf_rn(b2, v, __fmul_rn(__fmul_rn(omb2, g), g));
    a.m[e] = m;
    a.v[e] = v;
    // (explicitly rounded: the peer-exchange Adam, xg_dp.cu, must match bit for bit)
    a.p[e] = __fsub_rn(a.p[e], __fmul_rn(lrf[f], __fdiv_rn(__fdiv_rn(m, bc1), __fadd_rn(__fsqrt_rn(__fdiv_rn(v, bc2)), eps))));
  }
}

// The same update 4 elements per thread with 16-byte loads / stores (begin a
// multiple of 4, buffers 16-byte aligned): 4x the bytes in flight per
// thread.  Per element the arithmetic is k_adam's, so results are identical.
__device__ __forceinline__ void adam_one(float& p, float& m, float& v, float g, float lr, float b1, float b2,
                                         float omb1, float omb2, float bc1, float bc2, float eps) {
  m = __fmaf_rn(b1, m, __fmul_rn(omb1, g));
  v = __fmaf_rn(b2, v, __fmul_rn(__fmul_rn(omb2, g), g));
  p = __fsub_rn(p, __fmul_rn(lr, __fdiv_rn(__fdiv_rn(m, bc1), __fadd_rn(__fsqrt_rn(__fdiv_rn(v, bc2)), eps))));
}

__global__ void k_adam4(AdamArgs a) {
  const uint32_t bad = a.status ? (a.status[0] >> XG_ST_GRAD_NONFINITE_SHIFT) & 0x1f : 0u;
  const float b1 = (float)a.b1, b2 = (float)a.b2, omb1 = (float)(1.0 - a.b1), omb2 = (float)(1.0 - a.b2);
  const float bc1 = (float)a.bc1, bc2 = (float)a.bc2, eps = (float)a.eps;
  float lrf[kFields];
#pragma unroll
  for (int k = 0; k < kFields; ++k) lrf[k] = (float)a.lr[k];
  const long long v0 = a.begin >> 2, v1 = a.end >> 2;  // whole vectors; the < 4 tail elements below
  for (long long q = v0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; q < v1;
       q += (long long)gridDim.x * blockDim.x) {
    const long long e0 = q << 2;
    const float4 g4 = reinterpret_cast<const float4*>(a.g)[q];
    float4 m4 = reinterpret_cast<const float4*>(a.m)[q];
    float4 w4 = reinterpret_cast<const float4*>(a.v)[q];
    float4 p4 = reinterpret_cast<const float4*>(a.p)[q];
    float* pp = &p4.x;
    float* mm = &m4.x;
    float* ww = &w4.x;
    const float* gg = &g4.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const long long e = e0 + c;
      const int f = (e >= a.bound[0]) + (e >= a.bound[1]) + (e >= a.bound[2]) + (e >= a.bound[3]);
      if (bad & ((2u << f) - 1u)) continue;  // (unchanged values are written back)
      adam_one(pp[c], mm[c], ww[c], gg[c], lrf[f], b1, b2, omb1, omb2, bc1, bc2, eps);
    }
    reinterpret_cast<float4*>(a.m)[q] = m4;
    reinterpret_cast<float4*>(a.v)[q] = w4;
    reinterpret_cast<float4*>(a.p)[q] = p4;
  }
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long e = (v1 << 2) + t;
  if (e < a.end) {
    const int f = (e >= a.bound[0]) + (e >= a.bound[1]) + (e >= a.bound[2]) + (e >= a.bound[3]);
    if (!(bad & ((2u << f) - 1u))) {
      float p = a.p[e], m = a.m[e], v = a.v[e];
      adam_one(p, m, v, a.g[e], lrf[f], b1, b2, omb1, omb2, bc1, bc2, eps);
      a.m[e] = m;
      a.v[e] = v;
      a.p[e] = p;
    }
  }
}

// normalize_rotations (gaussians.py:234-235) after the update; skipped if
// any field diverged (the reference raises before renormalising).
__global__ void k_renorm(float* q_all, long long n, const uint32_t* status) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (status && ((status[0] >> XG_ST_GRAD_NONFINITE_SHIFT) & 0x1f)) return;
  float* q = q_all + 4 * i;  // 3n-float offset: not 16-byte aligned in general
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double nrm = sqrt(((w * w + x * x) + y * y) + z * z);
  q[0] = (float)(w / nrm);
  q[1] = (float)(x / nrm);
  q[2] = (float)(y / nrm);
  q[3] = (float)(z / nrm);
}

__device__ __forceinline__ double sigmoid64(double x) { return det_sigmoid(x); }

__global__ void k_densify_mark(const float* p, long long n, Layout L, const float* norm_sum,
                               const int32_t* obs, double gthr, double sthr, double pthr,
                               uint8_t* flags, uint32_t* counts) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  uint8_t fl = 0;
  if (i < n) {
    const int o = obs[i];
    const double avg = (double)norm_sum[i] / (double)(o > 1 ? o : 1);
    const bool high = avg >= gthr;
    const float* ls = p + L.off[2] + 3 * i;
    double mx = det_exp((double)ls[0]);
    mx = fmax(mx, det_exp((double)ls[1]));
    mx = fmax(mx, det_exp((double)ls[2]));
    const bool large = mx > sthr;
    const bool prune = sigmoid64((double)p[L.off[3] + i]) < pthr;
    const bool clone = high && !large && !prune;
    const bool split = high && large && !prune;
    fl = (uint8_t)(high | (large << 1) | (prune << 2) | (clone << 3) | (split << 4));
    flags[i] = fl;
  }
  const unsigned bp = __ballot_sync(0xffffffffu, fl & 4), bc = __ballot_sync(0xffffffffu, fl & 8),
                 bs = __ballot_sync(0xffffffffu, fl & 16);
  if (lane_id() == 0) {
    if (bp) atomicAdd(&counts[0], __popc(bp));
    if (bc) atomicAdd(&counts[1], __popc(bc));
    if (bs) atomicAdd(&counts[2], __popc(bs));
  }
}

// class masks for the scans: keep = !prune && !split (when growth is
// disabled split rows are kept, matching clone[:] = split[:] = False).
__global__ void k_class_masks(const uint8_t* flags, long long n, int allow, uint32_t* mk, uint32_t* mc,
                              uint32_t* ms) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t f = flags[i];
  const bool prune = f & 4;
  const bool clone = allow && (f & 8);
  const bool split = allow && (f & 16);
  mk[i] = (!prune && !split) ? 1u : 0u;
  mc[i] = clone ? 1u : 0u;
  ms[i] = split ? 1u : 0u;
}

__device__ __forceinline__ void rot_of(const float* q4, double* r) {
  double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
  const double nrm = sqrt(((w * w + x * x) + y * y) + z * z);
  w /= nrm; x /= nrm; y /= nrm; z /= nrm;
  r[0] = 1.0 - 2.0 * (y * y + z * z); r[1] = 2.0 * (x * y - w * z); r[2] = 2.0 * (x * z + w * y);
  r[3] = 2.0 * (x * y + w * z); r[4] = 1.0 - 2.0 * (x * x + z * z); r[5] = 2.0 * (y * z - w * x);
  r[6] = 2.0 * (x * z - w * y); r[7] = 2.0 * (y * z + w * x); r[8] = 1.0 - 2.0 * (x * x + y * y);
}

struct ApplyArgs {
  const float *p, *m, *v;
  long long n, n_new;
  Layout L, Ln;
  const uint32_t *mk, *mc, *ms;       // masks
  const uint32_t *sk, *sc, *ss;       // exclusive scans
  const uint32_t *tot;                // totals [keep, clone, split]
  const float* wgs;                   // world_grad_sum [n][3]
  const double* normals;              // [n_split][2][3]
  double log_split;
  float *np_, *nm, *nv;
};

__device__ __forceinline__ void copy_row(const ApplyArgs& a, long long src, long long dst, bool moments) {
  for (int f = 0; f < kFields; ++f) {
    const int w = a.L.width[f];
    const float* ps = a.p + a.L.off[f] + src * w;
    float* pd = a.np_ + a.Ln.off[f] + dst * w;
    for (int c = 0; c < w; ++c) pd[c] = ps[c];
    float* md = a.nm + a.Ln.off[f] + dst * w;
    float* vd = a.nv + a.Ln.off[f] + dst * w;
    if (moments) {
      const float* ms = a.m + a.L.off[f] + src * w;
      const float* vs = a.v + a.L.off[f] + src * w;
      for (int c = 0; c < w; ++c) md[c] = ms[c], vd[c] = vs[c];
    } else {
      for (int c = 0; c < w; ++c) md[c] = 0.f, vd[c] = 0.f;
    }
  }
}

__global__ void k_densify_apply(ApplyArgs a) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const long long n_keep = a.tot[0], n_clone = a.tot[1];
  if (a.mk[i]) copy_row(a, i, a.sk[i], true);
  if (a.mc[i]) {
    // clone nudged half a mean scale against the accumulated gradient
    const long long d = n_keep + a.sc[i];
    copy_row(a, i, d, false);
    const double gx = a.wgs[3 * i], gy = a.wgs[3 * i + 1], gz = a.wgs[3 * i + 2];
    const double nrm = sqrt(gx * gx + gy * gy + gz * gz);
    const float* ls = a.p + a.L.off[2] + 3 * i;
    const double step = 0.5 * ((det_exp((double)ls[0]) + det_exp((double)ls[1])) + det_exp((double)ls[2])) / 3.0;
    if (nrm > 0.0) {
      float* pd = a.np_ + a.Ln.off[0] + 3 * d;
      const float* ps = a.p + a.L.off[0] + 3 * i;
      pd[0] = (float)((double)ps[0] - step * (gx / nrm));
      pd[1] = (float)((double)ps[1] - step * (gy / nrm));
      pd[2] = (float)((double)ps[2] - step * (gz / nrm));
    }
  }
  if (a.ms[i]) {
    // two children sampling the parent's own distribution: mu + R (z * s)
    const long long k = a.ss[i];
    const long long d0 = n_keep + n_clone + 2 * k;
    double r[9];
    rot_of(a.p + a.L.off[1] + 4 * i, r);
    const float* ls = a.p + a.L.off[2] + 3 * i;
    const double s[3] = {det_exp((double)ls[0]), det_exp((double)ls[1]), det_exp((double)ls[2])};
    const float* ps = a.p + a.L.off[0] + 3 * i;
    for (int c = 0; c < 2; ++c) {
      const long long d = d0 + c;
      copy_row(a, i, d, false);
      const double* z = a.normals + 6 * k + 3 * c;
      const double lz[3] = {z[0] * s[0], z[1] * s[1], z[2] * s[2]};
      float* pd = a.np_ + a.Ln.off[0] + 3 * d;
      for (int row = 0; row < 3; ++row) {
        const double off = (r[3 * row] * lz[0] + r[3 * row + 1] * lz[1]) + r[3 * row + 2] * lz[2];
        pd[row] = (float)((double)ps[row] + off);
      }
      float* ld = a.np_ + a.Ln.off[2] + 3 * d;
      for (int q = 0; q < 3; ++q) ld[q] = (float)((double)ls[q] - a.log_split);
    }
  }
}

__global__ void k_totals(const uint32_t* sk, const uint32_t* mk, const uint32_t* sc, const uint32_t* mc,
                         const uint32_t* ss, const uint32_t* ms, long long n, uint32_t* tot) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    tot[0] = sk[n - 1] + mk[n - 1];
    tot[1] = sc[n - 1] + mc[n - 1];
    tot[2] = ss[n - 1] + ms[n - 1];
  }
}

}  // namespace
}  // namespace xg

using namespace xg;

extern "C" {

static xg_status adam_launch(float* params, const float* grads, float* exp_avg, float* exp_avg_sq, int64_t n,
                             int32_t n_features, const double* lr, double beta1, double beta2, double eps,
                             double bc1, double bc2, const uint32_t* status, int64_t begin, int64_t end,
                             cudaStream_t s) {
  if (!params || !grads || !exp_avg || !exp_avg_sq || !lr || n < 1 || n_features < 1 || begin < 0 ||
      end > n * (11 + n_features) || begin > end) {
    set_error_msg("xg_adam: invalid argument");
    return XG_ERR_INVALID;
  }
  if (begin == end) return XG_OK;
  AdamArgs a;
  a.p = params;
  a.g = grads;
  a.m = exp_avg;
  a.v = exp_avg_sq;
  a.n = n;
  a.bound[0] = 3 * n;
  a.bound[1] = 7 * n;
  a.bound[2] = 10 * n;
  a.bound[3] = 11 * n;
  a.begin = begin;
  a.end = end;
  for (int f = 0; f < kFields; ++f) a.lr[f] = lr[f];
  a.b1 = beta1;
  a.b2 = beta2;
  a.eps = eps;
  a.bc1 = bc1;
  a.bc2 = bc2;
  a.status = status;
  const int64_t cnt = end - begin;
  const bool vec = (begin & 3) == 0 && ((uintptr_t)params & 15) == 0 && ((uintptr_t)grads & 15) == 0 &&
                   ((uintptr_t)exp_avg & 15) == 0 && ((uintptr_t)exp_avg_sq & 15) == 0;
  int grid = div_up(vec ? (cnt + 3) / 4 : cnt, 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (vec) {
    k_adam4<<<grid, 256, 0, s>>>(a);
    return check_launch("k_adam4");
  }
  k_adam<<<grid, 256, 0, s>>>(a);
  return check_launch("k_adam");
}

xg_status xg_adam(float* params, const float* grads, float* exp_avg, float* exp_avg_sq, int64_t n,
                  int32_t n_features, const double* lr, double beta1, double beta2, double eps,
                  double bc1, double bc2, const uint32_t* status, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  xg_status st = adam_launch(params, grads, exp_avg, exp_avg_sq, n, n_features, lr, beta1, beta2, eps, bc1,
                             bc2, status, 0, n * (11 + n_features), s);
  if (st != XG_OK) return st;
  return xg_adam_renorm(params, n, n_features, status, stream);
}

xg_status xg_adam_range(float* params, const float* grads, float* exp_avg, float* exp_avg_sq, int64_t n,
                        int32_t n_features, const double* lr, double beta1, double beta2, double eps,
                        double bc1, double bc2, const uint32_t* status, int64_t elem_begin, int64_t elem_end,
                        void* stream) {
  return adam_launch(params, grads, exp_avg, exp_avg_sq, n, n_features, lr, beta1, beta2, eps, bc1, bc2,
                     status, elem_begin, elem_end, (cudaStream_t)stream);
}

xg_status xg_adam_renorm(float* params, int64_t n, int32_t n_features, const uint32_t* status, void* stream) {
  if (!params || n < 1) {
    set_error_msg("xg_adam_renorm: invalid argument");
    return XG_ERR_INVALID;
  }
  (void)n_features;
  k_renorm<<<div_up(n, 256), 256, 0, (cudaStream_t)stream>>>(params + 3 * n, n, status);
  return check_launch("k_renorm");
}

xg_status xg_densify_mark(const float* params, int64_t n, int32_t n_features, const float* norm_sum,
                          const int32_t* obs_count, double grad_threshold, double size_threshold,
                          double prune_opacity, uint8_t* flags, uint32_t* counts, void* stream) {
  if (!params || !norm_sum || !obs_count || !flags || !counts || n < 1) {
    set_error_msg("xg_densify_mark: invalid argument");
    return XG_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(counts, 0, 4 * sizeof(uint32_t), s);
  k_densify_mark<<<div_up(n, 128), 128, 0, s>>>(params, n, make_layout(n, n_features), norm_sum,
                                                obs_count, grad_threshold, size_threshold,
                                                prune_opacity, flags, counts);
  return check_launch("k_densify_mark");
}

xg_status xg_densify_apply(const float* params, const float* exp_avg, const float* exp_avg_sq,
                           int64_t n, int32_t n_features, const uint8_t* flags,
                           const float* world_grad_sum, const double* split_normals,
                           double log_split_factor, int32_t allow_growth, float* new_params,
                           float* new_exp_avg, float* new_exp_avg_sq, int64_t n_new,
                           uint32_t* scratch, void* stream) {
  if (!params || !exp_avg || !exp_avg_sq || !flags || !world_grad_sum || !new_params ||
      !new_exp_avg || !new_exp_avg_sq || !scratch || n < 1 || n_new < 1) {
    set_error_msg("xg_densify_apply: invalid argument");
    return XG_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  // scratch layout: 3 masks, 3 scans (n each), 3 totals, then scan workspace
  uint32_t* mk = scratch;
  uint32_t* mc = mk + n;
  uint32_t* ms = mc + n;
  uint32_t* sk = ms + n;
  uint32_t* sc = sk + n;
  uint32_t* ss = sc + n;
  uint32_t* tot = ss + n;
  void* sws = (void*)(((uintptr_t)(tot + 4) + 255) & ~(uintptr_t)255);
  const size_t sws_bytes = scan_workspace_bytes(n);
  k_class_masks<<<div_up(n, 256), 256, 0, s>>>(flags, n, allow_growth, mk, mc, ms);
  xg_status st = check_launch("k_class_masks");
  if (st != XG_OK) return st;
  if ((st = scan_u32(mk, nullptr, sk, n, nullptr, n, nullptr, sws, sws_bytes, s)) != XG_OK) return st;
  if ((st = scan_u32(mc, nullptr, sc, n, nullptr, n, nullptr, sws, sws_bytes, s)) != XG_OK) return st;
  if ((st = scan_u32(ms, nullptr, ss, n, nullptr, n, nullptr, sws, sws_bytes, s)) != XG_OK) return st;
  k_totals<<<1, 32, 0, s>>>(sk, mk, sc, mc, ss, ms, n, tot);
  ApplyArgs a;
  a.p = params;
  a.m = exp_avg;
  a.v = exp_avg_sq;
  a.n = n;
  a.n_new = n_new;
  a.L = make_layout(n, n_features);
  a.Ln = make_layout(n_new, n_features);
  a.mk = mk; a.mc = mc; a.ms = ms;
  a.sk = sk; a.sc = sc; a.ss = ss;
  a.tot = tot;
  a.wgs = world_grad_sum;
  a.normals = split_normals;
  a.log_split = log_split_factor;
  a.np_ = new_params;
  a.nm = new_exp_avg;
  a.nv = new_exp_avg_sq;
  k_densify_apply<<<div_up(n, 128), 128, 0, s>>>(a);
  return check_launch("k_densify_apply");
}

}  // extern "C"
