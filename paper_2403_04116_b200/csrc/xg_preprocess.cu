// K1 (projection / culling / tile rects) and K4b (per-Gaussian chain rule).
//
// One thread per Gaussian, float64 arithmetic throughout, compiled with
// -fmad=false so every product and sum rounds exactly as written (the
// oracle in oracle/xg_oracle.c performs the same operations in the same
// order): radii, tile rects and depth keys are bit-reproducible, and the
// float64 path sidesteps the float32 eigenvalue cancellation documented in
// SURVEY.md 7 ("hard parts" 1).  Per-Gaussian work is ~300 DFLOP, i.e. a
// few microseconds for 1M Gaussians, far from any roofline that matters.
#include <math.h>

#include "xg_internal.cuh"

namespace xg {

struct Cam {
  double r[9], t[3], f, cx, cy, near_plane;
  int w, h, ntx, nty;
};

__host__ static Cam make_cam(const xg_camera& c) {
  Cam k;
  for (int i = 0; i < 9; ++i) k.r[i] = c.rot[i];
  for (int i = 0; i < 3; ++i) k.t[i] = c.trans[i];
  k.f = c.focal;
  k.cx = c.cx;
  k.cy = c.cy;
  k.near_plane = c.near_plane;
  k.w = c.width;
  k.h = c.height;
  k.ntx = tiles_x(c);
  k.nty = tiles_y(c);
  return k;
}

struct CloudPtrs {
  const float* pos;
  const float* rot;
  const float* logs;
  const float* raw;
  const float* feat;
  const float* basis;
  const float* inten_pre;  // optional precomputed sigmoid(F . lambda) (xg_cloud.intensities)
  const double* inv;       // optional [N][8] view invariants (xg_cloud.invariants)
  long long n;
  int nf;
};

__host__ static CloudPtrs make_cloud(const xg_cloud& c) {
  CloudPtrs p;
  long long n = c.n;
  p.pos = c.params;
  p.rot = p.pos + 3 * n;
  p.logs = p.rot + 4 * n;
  p.raw = p.logs + 3 * n;
  p.feat = p.raw + n;
  p.basis = c.basis;
  p.inten_pre = c.intensities;
  p.inv = c.invariants;
  p.n = n;
  p.nf = c.n_features;
  return p;
}

// Everything project_splats derives for one Gaussian (frontend.py:116-158).
struct Proj {
  double t[3];   // camera-frame centre
  double u[2];   // pixel mean
  double rot[9]; // R(q/|q|)
  double s[3];   // exp(log_scale)
  double u2[6];  // J2 W (2x3)
  double sig3[6];  // Sigma3 xx xy xz yy yz zz
  double aa, bb, cc, det;
  double radius;
  bool visible;  // t_z > near
  bool zero_q;
};

// R(q/|q|), gaussians.py:55-68.
__device__ __forceinline__ bool quat_rot(const float* q4, double* r, double* qn) {
  double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
  double nrm = sqrt(((w * w + x * x) + y * y) + z * z);
  if (nrm == 0.0) return false;
  w = w / nrm;
  x = x / nrm;
  y = y / nrm;
  z = z / nrm;
  if (qn) {
    qn[0] = w; qn[1] = x; qn[2] = y; qn[3] = z; qn[4] = nrm;
  }
  r[0] = 1.0 - 2.0 * (y * y + z * z);
  r[1] = 2.0 * (x * y - w * z);
  r[2] = 2.0 * (x * z + w * y);
  r[3] = 2.0 * (x * y + w * z);
  r[4] = 1.0 - 2.0 * (x * x + z * z);
  r[5] = 2.0 * (y * z - w * x);
  r[6] = 2.0 * (x * z - w * y);
  r[7] = 2.0 * (y * z + w * x);
  r[8] = 1.0 - 2.0 * (x * x + y * y);
  return true;
}

// M = R diag(e^s); Sigma3 = M M^T (frontend.py:127-128)
__device__ __forceinline__ void sigma3(const CloudPtrs& c, long long i, const double* rot, double* s, double* sig3) {
  for (int a = 0; a < 3; ++a) s[a] = det_exp((double)c.logs[3 * i + a]);
  double m[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) m[3 * a + b] = rot[3 * a + b] * s[b];
  int q = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = a; b < 3; ++b)
      sig3[q++] = (m[3 * a] * m[3 * b] + m[3 * a + 1] * m[3 * b + 1]) + m[3 * a + 2] * m[3 * b + 2];
}

__device__ __forceinline__ void project_one(const CloudPtrs& c, const Cam& k, long long i, Proj& p,
                                            bool use_inv = false) {
  const double px = c.pos[3 * i], py = c.pos[3 * i + 1], pz = c.pos[3 * i + 2];
  // t = W mu + T (frontend.py:116).  The reference evaluates positions @ W^T
  // through BLAS dgemm, which accumulates as fma(w2, z, fma(w1, y, w0 x));
  // the same rounding keeps t_z - and so the depth order at exact real ties
  // (symmetric lattice views) - identical to the reference's.
  for (int a = 0; a < 3; ++a)
    p.t[a] = fma(k.r[3 * a + 2], pz, fma(k.r[3 * a + 1], py, k.r[3 * a] * px)) + k.t[a];
  p.visible = p.t[2] > k.near_plane;  // frontend.py:117
  p.zero_q = false;
  if (!p.visible) return;
  const double tz = p.t[2];
  p.u[0] = (k.f * p.t[0]) / tz + k.cx;  // frontend.py:122
  p.u[1] = (k.f * p.t[1]) / tz + k.cy;
  if (use_inv) {  // view-invariant cache (xg_view_invariants): the same numbers, computed once
    const double* v = c.inv + 8 * i;
    if (v[7] != 0.0) {
      p.zero_q = true;
      return;
    }
    for (int a = 0; a < 6; ++a) p.sig3[a] = v[a];
  } else {
    if (!quat_rot(c.rot + 4 * i, p.rot, nullptr)) {
      p.zero_q = true;
      return;
    }
    sigma3(c, i, p.rot, p.s, p.sig3);
  }
  // J2 (pixel units, no clamping; frontend.py:197-205) and U2 = J2 W (:129)
  const double j00 = k.f / tz;
  const double j02 = (-k.f * p.t[0]) / (tz * tz);
  const double j12 = (-k.f * p.t[1]) / (tz * tz);
  for (int b = 0; b < 3; ++b) {
    p.u2[b] = j00 * k.r[b] + j02 * k.r[6 + b];
    p.u2[3 + b] = j00 * k.r[3 + b] + j12 * k.r[6 + b];
  }
  // cov = U2 Sigma3 U2^T (:130) via tmp = U2 Sigma3
  double S[9] = {p.sig3[0], p.sig3[1], p.sig3[2], p.sig3[1], p.sig3[3],
                 p.sig3[4], p.sig3[2], p.sig3[4], p.sig3[5]};
  double tmp[6];
  for (int r = 0; r < 2; ++r)
    for (int b = 0; b < 3; ++b)
      tmp[3 * r + b] = (p.u2[3 * r] * S[b] + p.u2[3 * r + 1] * S[3 + b]) + p.u2[3 * r + 2] * S[6 + b];
  const double c00 = (tmp[0] * p.u2[0] + tmp[1] * p.u2[1]) + tmp[2] * p.u2[2];
  const double c01 = (tmp[0] * p.u2[3] + tmp[1] * p.u2[4]) + tmp[2] * p.u2[5];
  const double c11 = (tmp[3] * p.u2[3] + tmp[4] * p.u2[4]) + tmp[5] * p.u2[5];
  p.aa = c00 + XG_COV2_LOWPASS;  // :131-133
  p.bb = c01;
  p.cc = c11 + XG_COV2_LOWPASS;
  p.det = p.aa * p.cc - p.bb * p.bb;  // :134
  // r = 7.5 sqrt(lambda_max), lambda_max = mid + sqrt(max(mid^2 - det, 0)) (:139-141)
  const double mid = 0.5 * (p.aa + p.cc);
  const double disc = mid * mid - p.det;
  const double lam = mid + sqrt(disc > 0.0 ? disc : 0.0);
  p.radius = XG_CUTOFF_SIGMA * sqrt(lam);
}

__device__ __forceinline__ double intensity_of(const CloudPtrs& c, long long i, bool* finite) {
  double acc = 0.0;
  bool ok = true;
  for (int j = 0; j < c.nf; ++j) {
    const double f = c.feat[(long long)c.nf * i + j];
    const double b = c.basis[j];
    ok = ok && isfinite(f) && isfinite(b);
    acc = acc + f * b;
  }
  *finite = ok;
  return det_sigmoid(acc);
}

#ifndef XG_PRE_MIN_CTAS
#define XG_PRE_MIN_CTAS 1
#endif
#ifndef XG_PRE_BWD_MIN_CTAS
#define XG_PRE_BWD_MIN_CTAS 1
#endif
__global__ void __launch_bounds__(128, XG_PRE_MIN_CTAS) k_preprocess(CloudPtrs c, Cam k, xg_splats sp,
                                                                     xg_splat_extras ex) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned status = 0;
  bool active = false;
  if (i < c.n) {
    Proj p;
    const bool use_inv = c.inv != nullptr;
    project_one(c, k, i, p, use_inv);
    if (c.inten_pre) {  // view-independent: computed once per cloud (xg_intensities)
      if (sp.inten != c.inten_pre) sp.inten[i] = c.inten_pre[i];
    } else {
      bool finite;
      const double inten = intensity_of(c, i, &finite);
      sp.inten[i] = (float)inten;
      if (!finite) status |= XG_ST_NONFINITE_FEAT;
    }
    uint32_t ntiles = 0;
    unsigned long long key = ~0ull;
    if (p.visible && p.zero_q) status |= XG_ST_ZERO_QUAT;
    if (p.visible && !p.zero_q) {
      if (!(p.det > 0.0) || !isfinite(p.det)) status |= XG_ST_DEGENERATE;
      // tile rect (frontend.py:143-148): floor((u -+ r) / 16), clamped
      const double fx0 = floor((p.u[0] - p.radius) / kTile);
      const double fx1 = floor((p.u[0] + p.radius) / kTile);
      const double fy0 = floor((p.u[1] - p.radius) / kTile);
      const double fy1 = floor((p.u[1] + p.radius) / kTile);
      const double tx0 = fx0 > 0.0 ? fx0 : 0.0;
      const double tx1 = fx1 < (double)(k.ntx - 1) ? fx1 : (double)(k.ntx - 1);
      const double ty0 = fy0 > 0.0 ? fy0 : 0.0;
      const double ty1 = fy1 < (double)(k.nty - 1) ? fy1 : (double)(k.nty - 1);
      if (p.det > 0.0 && tx0 <= tx1 && ty0 <= ty1) {
        active = true;
        const int ix0 = (int)tx0, ix1 = (int)tx1, iy0 = (int)ty0, iy1 = (int)ty1;
        ntiles = (uint32_t)((ix1 - ix0 + 1) * (iy1 - iy0 + 1));
        key = (unsigned long long)__double_as_longlong(p.t[2]);  // t_z > near > 0: bit order = value order
        sp.rect[4 * i + 0] = (uint16_t)ix0;
        sp.rect[4 * i + 1] = (uint16_t)iy0;
        sp.rect[4 * i + 2] = (uint16_t)ix1;
        sp.rect[4 * i + 3] = (uint16_t)iy1;
        sp.mean2d[2 * i + 0] = p.u[0];
        sp.mean2d[2 * i + 1] = p.u[1];
        // conic = (cc, -bb, aa) / det (frontend.py:137) on the log2 scale:
        // p2 = -0.5 log2e (a dx^2 + c dy^2) - log2e b dx dy
        const double ca = p.cc / p.det, cb = -p.bb / p.det, cc = p.aa / p.det;
        const double alpha = use_inv ? c.inv[8 * i + 6] : det_sigmoid((double)c.raw[i]);
        float4 cf;
        cf.x = (float)(-0.5 * kLog2e * ca);
        cf.y = (float)(-kLog2e * cb);
        cf.z = (float)(-0.5 * kLog2e * cc);
        cf.w = (float)alpha;
        reinterpret_cast<float4*>(sp.coef)[i] = cf;
        if (ex.cov2d) {
          ex.cov2d[3 * i] = p.aa; ex.cov2d[3 * i + 1] = p.bb; ex.cov2d[3 * i + 2] = p.cc;
        }
        if (ex.conic) {
          ex.conic[3 * i] = ca; ex.conic[3 * i + 1] = cb; ex.conic[3 * i + 2] = cc;
        }
        if (ex.depth) ex.depth[i] = p.t[2];
        if (ex.t_cam) {
          ex.t_cam[3 * i] = p.t[0]; ex.t_cam[3 * i + 1] = p.t[1]; ex.t_cam[3 * i + 2] = p.t[2];
        }
        if (ex.radius) ex.radius[i] = p.radius;
        if (ex.opacity) ex.opacity[i] = alpha;
      }
    }
    sp.n_tiles[i] = ntiles;
    reinterpret_cast<unsigned long long*>(sp.depth_key)[i] = key;
  }
  // warp-aggregated counters
  const unsigned act = __ballot_sync(0xffffffffu, active);
  const unsigned st = __reduce_or_sync(0xffffffffu, status);
  if (lane_id() == 0) {
    if (act) atomicAdd(&sp.counters[XG_CTR_ACTIVE], (unsigned)__popc(act));
    if (st) atomicOr(&sp.counters[XG_CTR_STATUS], st);
  }
}

__global__ void k_view_invariants(CloudPtrs c, double* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c.n) return;
  double rot[9], s[3], sig3[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const bool ok = quat_rot(c.rot + 4 * i, rot, nullptr);
  if (ok) sigma3(c, i, rot, s, sig3);
  double* o = out + 8 * i;
  for (int a = 0; a < 6; ++a) o[a] = sig3[a];
  o[6] = det_sigmoid((double)c.raw[i]);
  o[7] = ok ? 0.0 : 1.0;
}

__global__ void k_intensities(CloudPtrs c, float* out, uint32_t* counters) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool finite = true;
  if (i < c.n) out[i] = (float)intensity_of(c, i, &finite);
  const unsigned bad = __ballot_sync(0xffffffffu, !finite);
  if (bad && lane_id() == 0 && counters) atomicOr(&counters[XG_CTR_STATUS], XG_ST_NONFINITE_FEAT);
}

// ---------------------------------------------------------------------------
// K4b: backward.py:61-158 for one active Gaussian.
// ---------------------------------------------------------------------------
struct BwdOut {
  float* grads;  // flat
  float* screen_norms;
  uint8_t* visible;
  float* norm_sum;
  int32_t* obs_count;
  float* world_grad_sum;
  double* g_mean;
  double* g_conic;
  double* g_int;
  double* g_alpha;
  uint32_t* counters;
};

__global__ void __launch_bounds__(128, XG_PRE_BWD_MIN_CTAS) k_preprocess_bwd(CloudPtrs c, Cam k, xg_splats sp, const float* __restrict__ acc,
                                 BwdOut o) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bad = 0;
  if (i < c.n) {
    const long long n = c.n;
    float* g_pos = o.grads + 3 * i;
    float* g_rot = o.grads + 3 * n + 4 * i;
    float* g_ls = o.grads + 7 * n + 3 * i;
    float* g_raw = o.grads + 10 * n + i;
    float* g_feat = o.grads + 11 * n + (long long)c.nf * i;
    const bool active = sp.n_tiles[i] != 0;
    if (!active) {
      for (int a = 0; a < 3; ++a) g_pos[a] = 0.f, g_ls[a] = 0.f;
      for (int a = 0; a < 4; ++a) g_rot[a] = 0.f;
      *g_raw = 0.f;
      for (int j = 0; j < c.nf; ++j) g_feat[j] = 0.f;
      if (o.screen_norms) o.screen_norms[i] = 0.f;
      if (o.visible) o.visible[i] = 0;
      if (o.g_mean) { o.g_mean[2 * i] = 0.0; o.g_mean[2 * i + 1] = 0.0; }
      if (o.g_conic) { o.g_conic[3 * i] = 0.0; o.g_conic[3 * i + 1] = 0.0; o.g_conic[3 * i + 2] = 0.0; }
      if (o.g_int) o.g_int[i] = 0.0;
      if (o.g_alpha) o.g_alpha[i] = 0.0;
    } else {
      // every global read this thread needs issued before the projection's
      // float64 chain (their latency overlaps it instead of following it):
      // the replay's accumulators, the splat's coefficients, the opacity,
      // the features (intensity) and the DensifyStats being accumulated
      const float4 a0 = reinterpret_cast<const float4*>(acc)[2 * i];
      const float4 a1 = reinterpret_cast<const float4*>(acc)[2 * i + 1];
      const float4 cf = reinterpret_cast<const float4*>(sp.coef)[i];
      const float raw_i = c.raw[i];
      bool finite;
      const double it = intensity_of(c, i, &finite);
      const float ns_prev = o.norm_sum ? o.norm_sum[i] : 0.f;
      const int32_t oc_prev = o.obs_count ? o.obs_count[i] : 0;
      Proj p;
      project_one(c, k, i, p);
      // kernel accumulators -> reference kernel outputs (xgauss.h, K4a):
      // sum G (2 A2 dx + B2 dy) = 2 A2 sum G dx + B2 sum G dy, and the mean
      // gradient is -ln2 times that (p2 = power * log2 e, dx = px - mx)
      const double sdx = a0.x, sdy = a0.y;
      const double gmx = -kLn2 * (2.0 * (double)cf.x * sdx + (double)cf.y * sdy);
      const double gmy = -kLn2 * ((double)cf.y * sdx + 2.0 * (double)cf.z * sdy);
      const double gca = -0.5 * (double)a0.z;
      const double gcb = -(double)a0.w;
      const double gcc = -0.5 * (double)a1.x;
      const double gint = (double)a1.y;
      const double gpow = (double)a1.z;
      const double alpha = det_sigmoid((double)raw_i);
      const double galpha = alpha > 0.0 ? gpow / alpha : 0.0;  // sum dsigma*dens
      if (o.g_mean) { o.g_mean[2 * i] = gmx; o.g_mean[2 * i + 1] = gmy; }
      if (o.g_conic) { o.g_conic[3 * i] = gca; o.g_conic[3 * i + 1] = gcb; o.g_conic[3 * i + 2] = gcc; }
      if (o.g_int) o.g_int[i] = gint;
      if (o.g_alpha) o.g_alpha[i] = galpha;

      // conic -> cov2d: g2 = -K Gt K (backward.py:66-77)
      const double ka = p.cc / p.det, kb = -p.bb / p.det, kc = p.aa / p.det;
      const double ga = gca, gb = 0.5 * gcb, gc = gcc;
      // K Gt
      const double m00 = ka * ga + kb * gb, m01 = ka * gb + kb * gc;
      const double m10 = kb * ga + kc * gb, m11 = kb * gb + kc * gc;
      // -(K Gt) K
      const double g00 = -(m00 * ka + m01 * kb), g01 = -(m00 * kb + m01 * kc);
      const double g10 = -(m10 * ka + m11 * kb), g11 = -(m10 * kb + m11 * kc);
      const double G2[4] = {g00, g01, g10, g11};
      const double* U = p.u2;  // 2x3
      double S[9] = {p.sig3[0], p.sig3[1], p.sig3[2], p.sig3[1], p.sig3[3],
                     p.sig3[4], p.sig3[2], p.sig3[4], p.sig3[5]};
      // g_sigma3 = U^T G2 U (:90)
      double GU[6];
      for (int r = 0; r < 2; ++r)
        for (int b = 0; b < 3; ++b) GU[3 * r + b] = G2[2 * r] * U[b] + G2[2 * r + 1] * U[3 + b];
      double gS[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) gS[3 * a + b] = U[a] * GU[b] + U[3 + a] * GU[3 + b];
      // g_u2 = 2 G2 U Sigma3 (:91)
      double gU2[6];
      for (int r = 0; r < 2; ++r)
        for (int b = 0; b < 3; ++b)
          gU2[3 * r + b] =
              2.0 * ((GU[3 * r] * S[b] + GU[3 * r + 1] * S[3 + b]) + GU[3 * r + 2] * S[6 + b]);
      // g_j2 = g_u2 W^T (:92)
      double gJ[6];
      for (int r = 0; r < 2; ++r)
        for (int b = 0; b < 3; ++b)
          gJ[3 * r + b] = (gU2[3 * r] * k.r[3 * b] + gU2[3 * r + 1] * k.r[3 * b + 1]) +
                          gU2[3 * r + 2] * k.r[3 * b + 2];
      // g_t (:96-103)
      const double tx = p.t[0], ty = p.t[1], tz = p.t[2], f = k.f;
      const double tz2 = tz * tz, tz3 = tz2 * tz;
      double gt[3];
      gt[0] = gmx * f / tz - gJ[2] * f / tz2;
      gt[1] = gmy * f / tz - gJ[5] * f / tz2;
      gt[2] = -f * (gmx * tx + gmy * ty) / tz2 - f * (gJ[0] + gJ[4]) / tz2 +
              2.0 * f * (gJ[2] * tx + gJ[5] * ty) / tz3;
      // g_pos = g_t W (:104)
      double gp[3];
      for (int b = 0; b < 3; ++b) gp[b] = (gt[0] * k.r[b] + gt[1] * k.r[3 + b]) + gt[2] * k.r[6 + b];
      // g_M = 2 gS M ; g_log_s ; g_R (:106-108)
      double m[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m[3 * a + b] = p.rot[3 * a + b] * p.s[b];
      double gM[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          gM[3 * a + b] = 2.0 * ((gS[3 * a] * m[b] + gS[3 * a + 1] * m[3 + b]) + gS[3 * a + 2] * m[6 + b]);
      double gls[3], gR[9];
      for (int b = 0; b < 3; ++b) {
        gls[b] = ((p.rot[b] * gM[b] + p.rot[3 + b] * gM[3 + b]) + p.rot[6 + b] * gM[6 + b]) * p.s[b];
        for (int a = 0; a < 3; ++a) gR[3 * a + b] = gM[3 * a + b] * p.s[b];
      }
      // quaternion chain through R(q/|q|) (:127-158)
      double r9[9], qn[5];
      quat_rot(c.rot + 4 * i, r9, qn);
      const double qw = qn[0], qx = qn[1], qy = qn[2], qz = qn[3], nrm = qn[4];
      const double* g = gR;
      double gu[4];
      gu[0] = 2.0 * (-g[1] * qz + g[2] * qy + g[3] * qz - g[5] * qx - g[6] * qy + g[7] * qx);
      gu[1] = 2.0 * (g[1] * qy + g[2] * qz + g[3] * qy - 2.0 * g[4] * qx - g[5] * qw + g[6] * qz +
                     g[7] * qw - 2.0 * g[8] * qx);
      gu[2] = 2.0 * (-2.0 * g[0] * qy + g[1] * qx + g[2] * qw + g[3] * qx + g[5] * qz - g[6] * qw +
                     g[7] * qz - 2.0 * g[8] * qy);
      gu[3] = 2.0 * (-2.0 * g[0] * qz - g[1] * qw + g[2] * qx + g[3] * qw - 2.0 * g[4] * qz +
                     g[5] * qy + g[6] * qx + g[7] * qy);
      const double inner = qw * gu[0] + qx * gu[1] + qy * gu[2] + qz * gu[3];
      const double qv[4] = {qw, qx, qy, qz};
      // features / opacity (:112-115)
      const double gf = gint * it * (1.0 - it);
      const double graw = gpow * (1.0 - alpha);  // = g_alpha * alpha * (1 - alpha)

      float fv;
      bool ok;
      ok = true;
      for (int a = 0; a < 3; ++a) { fv = (float)gp[a]; g_pos[a] = fv; ok = ok && isfinite(fv); }
      if (!ok) bad |= 1u << 0;
      ok = true;
      for (int a = 0; a < 4; ++a) { fv = (float)((gu[a] - qv[a] * inner) / nrm); g_rot[a] = fv; ok = ok && isfinite(fv); }
      if (!ok) bad |= 1u << 1;
      ok = true;
      for (int a = 0; a < 3; ++a) { fv = (float)gls[a]; g_ls[a] = fv; ok = ok && isfinite(fv); }
      if (!ok) bad |= 1u << 2;
      fv = (float)graw;
      *g_raw = fv;
      if (!isfinite(fv)) bad |= 1u << 3;
      ok = true;
      for (int j = 0; j < c.nf; ++j) { fv = (float)(gf * (double)c.basis[j]); g_feat[j] = fv; ok = ok && isfinite(fv); }
      if (!ok) bad |= 1u << 4;

      const float sn = (float)hypot(gmx, gmy);
      if (o.screen_norms) o.screen_norms[i] = sn;
      if (o.visible) o.visible[i] = 1;
      if (o.norm_sum) o.norm_sum[i] = ns_prev + sn;
      if (o.obs_count) o.obs_count[i] = oc_prev + 1;
      if (o.world_grad_sum)
        for (int a = 0; a < 3; ++a) o.world_grad_sum[3 * i + a] += (float)gp[a];
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && lane_id() == 0 && o.counters) {
    atomicOr(&o.counters[XG_CTR_STATUS], bad << XG_ST_GRAD_NONFINITE_SHIFT);
    // and the caller's sticky word, which gates its Adam (xg_adam status)
    atomicOr(&o.counters[XG_CTR_STICKY], bad << XG_ST_GRAD_NONFINITE_SHIFT);
  }
}

__global__ void k_check_finite(const float* __restrict__ g, long long n, int nf, long long begin, long long end,
                               uint32_t* counters) {
  const long long total = n * (11 + nf);
  const long long bounds[5] = {3 * n, 7 * n, 10 * n, 11 * n, total};
  unsigned bad = 0;
  for (long long e = begin + (long long)blockIdx.x * blockDim.x + threadIdx.x; e < end;
       e += (long long)gridDim.x * blockDim.x) {
    if (!isfinite(g[e])) {
      int f = 0;
      while (e >= bounds[f]) ++f;
      bad |= 1u << f;
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && lane_id() == 0) atomicOr(&counters[XG_CTR_STATUS], bad << XG_ST_GRAD_NONFINITE_SHIFT);
}

}  // namespace xg

using namespace xg;

extern "C" {

int32_t xg_tiles_x(const xg_camera* cam) { return cam ? tiles_x(*cam) : 0; }
int32_t xg_tiles_y(const xg_camera* cam) { return cam ? tiles_y(*cam) : 0; }

xg_status xg_preprocess_fwd(const xg_cloud* cloud, const xg_camera* cam, xg_splats* sp,
                            const xg_splat_extras* extras, void* stream) {
  if (!cloud || !cam || !sp || !cloud->params || !cloud->basis || cloud->n < 1 || !sp->mean2d ||
      !sp->coef || !sp->inten || !sp->rect || !sp->n_tiles || !sp->depth_key || !sp->counters ||
      cam->width < 1 || cam->height < 1) {
    set_error_msg("xg_preprocess_fwd: invalid argument");
    return XG_ERR_INVALID;
  }
  if (tiles_x(*cam) > 65535 || tiles_y(*cam) > 65535) {
    set_error_msg("xg_preprocess_fwd: detector too large for 16-bit tile coordinates");
    return XG_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(sp->counters, 0, XG_CTR_STICKY * sizeof(uint32_t), s);
  cudaMemsetAsync(sp->counters + XG_CTR_L1, 0, 2 * sizeof(uint32_t), s);  // the fused-L1 accumulator (double)
  xg_splat_extras ex = {};
  if (extras) ex = *extras;
  const int block = 128;
  k_preprocess<<<div_up(cloud->n, block), block, 0, s>>>(make_cloud(*cloud), make_cam(*cam), *sp, ex);
  return check_launch("k_preprocess");
}

xg_status xg_view_invariants(const xg_cloud* cloud, double* out, void* stream) {
  if (!cloud || !cloud->params || cloud->n < 0 || (cloud->n > 0 && !out)) {
    set_error_msg("xg_view_invariants: invalid argument");
    return XG_ERR_INVALID;
  }
  if (cloud->n == 0) return XG_OK;
  const int block = 256;
  k_view_invariants<<<div_up(cloud->n, block), block, 0, (cudaStream_t)stream>>>(make_cloud(*cloud), out);
  return check_launch("k_view_invariants");
}

xg_status xg_intensities(const xg_cloud* cloud, float* out, uint32_t* counters, void* stream) {
  if (!cloud || !cloud->params || !cloud->basis || !out || cloud->n < 1) {
    set_error_msg("xg_intensities: invalid argument");
    return XG_ERR_INVALID;
  }
  const int block = 128;
  k_intensities<<<div_up(cloud->n, block), block, 0, (cudaStream_t)stream>>>(make_cloud(*cloud), out,
                                                                             counters);
  return check_launch("k_intensities");
}

xg_status xg_preprocess_bwd(const xg_cloud* cloud, const xg_camera* cam, const xg_splats* sp,
                            const float* grad_acc, float* grads, float* screen_norms,
                            uint8_t* visible, float* norm_sum, int32_t* obs_count,
                            float* world_grad_sum, double* g_mean_out, double* g_conic_out,
                            double* g_int_out, double* g_alpha_out, void* stream) {
  if (!cloud || !cam || !sp || !grad_acc || !grads || !cloud->params || cloud->n < 1) {
    set_error_msg("xg_preprocess_bwd: invalid argument");
    return XG_ERR_INVALID;
  }
  BwdOut o{grads, screen_norms, visible, norm_sum, obs_count, world_grad_sum,
           g_mean_out, g_conic_out, g_int_out, g_alpha_out, sp->counters};
  const int block = 128;
  k_preprocess_bwd<<<div_up(cloud->n, block), block, 0, (cudaStream_t)stream>>>(
      make_cloud(*cloud), make_cam(*cam), *sp, grad_acc, o);
  return check_launch("k_preprocess_bwd");
}

xg_status xg_check_finite(const float* grads, int64_t n, int32_t n_features, uint32_t* counters,
                          void* stream) {
  if (!grads || !counters || n < 1) {
    set_error_msg("xg_check_finite: invalid argument");
    return XG_ERR_INVALID;
  }
  k_check_finite<<<296, 256, 0, (cudaStream_t)stream>>>(grads, n, n_features, 0, n * (11 + n_features),
                                                        counters);
  return check_launch("k_check_finite");
}

xg_status xg_check_finite_range(const float* grads, int64_t n, int32_t n_features, int64_t elem_begin,
                                int64_t elem_end, uint32_t* counters, void* stream) {
  if (!grads || !counters || n < 1 || elem_begin < 0 || elem_end > n * (11 + n_features) ||
      elem_begin > elem_end) {
    set_error_msg("xg_check_finite_range: invalid argument");
    return XG_ERR_INVALID;
  }
  if (elem_begin == elem_end) return XG_OK;
  k_check_finite<<<296, 256, 0, (cudaStream_t)stream>>>(grads, n, n_features, elem_begin, elem_end, counters);
  return check_launch("k_check_finite");
}

}  // extern "C"
