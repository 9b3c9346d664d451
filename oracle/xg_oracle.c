/*
 * xg_oracle.c - CPU restatement of the reference DRR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it, and never as the thing measured or shipped.
 *
 * It restates, in plain C, the algorithm of xsplat 0.1.0 (the reference,
 * /root/reference/pkg/src/xsplat) in the arithmetic the engine uses:
 *
 *   xgo_preprocess     rasterizer/frontend.py:111-158 (projection, near cull,
 *                      cov2D, conic, radius, tile rect) and
 *                      gaussians.py:47-69, 110-124, 222-232 - float64, every
 *                      product/sum in the order written (built with
 *                      -ffp-contract=off), so radii, rects and depth keys
 *                      are bit-identical to the engine's
 *   xgo_bin            frontend.py:160-173: entries sorted by (tile,
 *                      float64 depth, cloud index), tile ranges
 *   xgo_composite_fwd  rasterizer/_kernels.pyx:41-73 in float32 with the
 *                      engine's operation order; additionally reports
 *                      n_contrib / n_traversed per pixel and flags pixels
 *                      whose early-termination decision sits within float
 *                      noise of the 1e-4 floor ("ambiguous")
 *   xgo_composite_bwd  rasterizer/_kernels.pyx:106-177 gradient pass in
 *                      float64 (reference formula: suffix = acc - prefix -
 *                      contrib), on the float32 forward's decisions
 *
 * The deterministic exp (det_exp) is an independent copy of the same
 * algorithm the engine uses for per-Gaussian sigmoids and scales
 * (Cody-Waite + Taylor-13 Horner with fma), so both sides agree bit for bit.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define TILE 16
#define LOG2E 1.4426950408889634073599246810019
#define POWER_CUTOFF (-30.0)
#define FLOOR_F 1e-4f
#define CLAMP_F 0.99f
#define CUTOFF_SIGMA 7.5
#define LOWPASS 0.3

typedef struct {
  double rot[9];
  double trans[3];
  double focal, cx, cy, near_plane;
  int32_t width, height;
} ocam;

static double det_exp(double x) {
  if (!(x == x)) return x;
  if (x > 709.0) return INFINITY;
  if (x < -745.0) return 0.0;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  double kd = (double)(long long)(x * 1.44269504088896338700e+00 + (x >= 0 ? 0.5 : -0.5));
  double r = fma(-kd, ln2_hi, x);
  r = fma(-kd, ln2_lo, r);
  double p = 1.6059043836821614599e-10;
  p = fma(p, r, 2.0876756987868098979e-09);
  p = fma(p, r, 2.5052108385441718775e-08);
  p = fma(p, r, 2.7557319223985890653e-07);
  p = fma(p, r, 2.7557319223985890653e-06);
  p = fma(p, r, 2.4801587301587301587e-05);
  p = fma(p, r, 1.9841269841269841270e-04);
  p = fma(p, r, 1.3888888888888888889e-03);
  p = fma(p, r, 8.3333333333333333333e-03);
  p = fma(p, r, 4.1666666666666666667e-02);
  p = fma(p, r, 1.6666666666666666667e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  long long k = (long long)kd;
  long long k1 = k / 2, k2 = k - k1;
  union { double d; unsigned long long u; } s1, s2;
  s1.u = (unsigned long long)(k1 + 1023) << 52;
  s2.u = (unsigned long long)(k2 + 1023) << 52;
  return (p * s1.d) * s2.d;
}

/* gaussians.py:29-38 */
static double sigmoid(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + det_exp(-x));
  double e = det_exp(x);
  return e / (1.0 + e);
}

/* ------------------------------------------------------------------------ */
/* xgo_preprocess: status bits 1 zero quaternion, 2 degenerate, 4 non-finite
 * features (same meaning as the engine's XG_ST_*). */
int xgo_preprocess(int64_t n, int32_t nf, const float* params, const float* basis, const ocam* cam,
                   double* mean2d, float* coef, float* inten, int32_t* rect, int32_t* n_tiles,
                   uint64_t* depth_key, double* radius, double* conic, double* cov2d, double* depth,
                   double* tcam, double* opacity, int64_t* n_active) {
  const float* P = params;
  const float* Q = params + 3 * n;
  const float* LS = params + 7 * n;
  const float* RAW = params + 10 * n;
  const float* F = params + 11 * n;
  const int ntx = (cam->width + TILE - 1) / TILE, nty = (cam->height + TILE - 1) / TILE;
  const double* W = cam->rot;
  int status = 0;
  int64_t act = 0;
  for (int64_t i = 0; i < n; ++i) {
    /* intensity: sigmoid(F . lambda), gaussians.py:110-124 */
    double s = 0.0;
    int finite = 1;
    for (int j = 0; j < nf; ++j) {
      double f = F[nf * i + j], b = basis[j];
      if (!isfinite(f) || !isfinite(b)) finite = 0;
      s = s + f * b;
    }
    if (!finite) status |= 4;
    inten[i] = (float)sigmoid(s);
    n_tiles[i] = 0;
    depth_key[i] = ~(uint64_t)0;
    /* t = W mu + T, frontend.py:116 */
    /* the reference's BLAS dgemm accumulates fma(w2, z, fma(w1, y, w0 x)) */
    double px = P[3 * i], py = P[3 * i + 1], pz = P[3 * i + 2], t[3];
    for (int a = 0; a < 3; ++a) t[a] = fma(W[3 * a + 2], pz, fma(W[3 * a + 1], py, W[3 * a] * px)) + cam->trans[a];
    if (!(t[2] > cam->near_plane)) continue; /* :117 */
    double tz = t[2];
    double ux = (cam->focal * t[0]) / tz + cam->cx; /* :122 */
    double uy = (cam->focal * t[1]) / tz + cam->cy;
    /* R(q/|q|), gaussians.py:55-68 */
    double w = Q[4 * i], x = Q[4 * i + 1], y = Q[4 * i + 2], z = Q[4 * i + 3];
    double nq = sqrt(((w * w + x * x) + y * y) + z * z);
    if (nq == 0.0) { status |= 1; continue; }
    w = w / nq; x = x / nq; y = y / nq; z = z / nq;
    double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                   2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                   2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
    double sc[3];
    for (int a = 0; a < 3; ++a) sc[a] = det_exp((double)LS[3 * i + a]);
    /* Sigma3 = (R S)(R S)^T, frontend.py:127-128 */
    double M[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) M[3 * a + b] = R[3 * a + b] * sc[b];
    double S[9];
    for (int a = 0; a < 3; ++a)
      for (int b = a; b < 3; ++b) {
        double v = (M[3 * a] * M[3 * b] + M[3 * a + 1] * M[3 * b + 1]) + M[3 * a + 2] * M[3 * b + 2];
        S[3 * a + b] = v;
        S[3 * b + a] = v;
      }
    /* U2 = J2 W, J2 in pixel units without clamping (frontend.py:129,197-205) */
    double j00 = cam->focal / tz;
    double j02 = (-cam->focal * t[0]) / (tz * tz);
    double j12 = (-cam->focal * t[1]) / (tz * tz);
    double U[6];
    for (int b = 0; b < 3; ++b) {
      U[b] = j00 * W[b] + j02 * W[6 + b];
      U[3 + b] = j00 * W[3 + b] + j12 * W[6 + b];
    }
    /* cov = (U2 Sigma3) U2^T + 0.3 I, :130-133 */
    double T6[6];
    for (int r = 0; r < 2; ++r)
      for (int b = 0; b < 3; ++b)
        T6[3 * r + b] = (U[3 * r] * S[b] + U[3 * r + 1] * S[3 + b]) + U[3 * r + 2] * S[6 + b];
    double c00 = (T6[0] * U[0] + T6[1] * U[1]) + T6[2] * U[2];
    double c01 = (T6[0] * U[3] + T6[1] * U[4]) + T6[2] * U[5];
    double c11 = (T6[3] * U[3] + T6[4] * U[4]) + T6[5] * U[5];
    double aa = c00 + LOWPASS, bb = c01, cc = c11 + LOWPASS;
    double det = aa * cc - bb * bb; /* :134-136 */
    if (!(det > 0.0) || !isfinite(det)) { status |= 2; continue; }
    /* radius 7.5 sqrt(lambda_max), :139-141 */
    double mid = 0.5 * (aa + cc);
    double disc = mid * mid - det;
    double lam = mid + sqrt(disc > 0.0 ? disc : 0.0);
    double rad = CUTOFF_SIGMA * sqrt(lam);
    /* tile rect, :143-148 */
    double fx0 = floor((ux - rad) / TILE), fx1 = floor((ux + rad) / TILE);
    double fy0 = floor((uy - rad) / TILE), fy1 = floor((uy + rad) / TILE);
    double tx0 = fx0 > 0.0 ? fx0 : 0.0, tx1 = fx1 < (double)(ntx - 1) ? fx1 : (double)(ntx - 1);
    double ty0 = fy0 > 0.0 ? fy0 : 0.0, ty1 = fy1 < (double)(nty - 1) ? fy1 : (double)(nty - 1);
    if (!(tx0 <= tx1 && ty0 <= ty1)) continue; /* on-screen cull */
    ++act;
    int ix0 = (int)tx0, ix1 = (int)tx1, iy0 = (int)ty0, iy1 = (int)ty1;
    rect[4 * i] = ix0; rect[4 * i + 1] = iy0; rect[4 * i + 2] = ix1; rect[4 * i + 3] = iy1;
    n_tiles[i] = (ix1 - ix0 + 1) * (iy1 - iy0 + 1);
    memcpy(&depth_key[i], &tz, 8);
    mean2d[2 * i] = ux;
    mean2d[2 * i + 1] = uy;
    double ka = cc / det, kb = -bb / det, kc = aa / det; /* conic, :137 */
    double alpha = sigmoid((double)RAW[i]);
    coef[4 * i] = (float)(-0.5 * LOG2E * ka);
    coef[4 * i + 1] = (float)(-LOG2E * kb);
    coef[4 * i + 2] = (float)(-0.5 * LOG2E * kc);
    coef[4 * i + 3] = (float)alpha;
    if (radius) radius[i] = rad;
    if (conic) { conic[3 * i] = ka; conic[3 * i + 1] = kb; conic[3 * i + 2] = kc; }
    if (cov2d) { cov2d[3 * i] = aa; cov2d[3 * i + 1] = bb; cov2d[3 * i + 2] = cc; }
    if (depth) depth[i] = tz;
    if (tcam) { tcam[3 * i] = t[0]; tcam[3 * i + 1] = t[1]; tcam[3 * i + 2] = t[2]; }
    if (opacity) opacity[i] = alpha;
  }
  *n_active = act;
  return status;
}

/* ------------------------------------------------------------------------ */
typedef struct { uint64_t key; uint32_t idx; } kv;

static int cmp_kv(const void* a, const void* b) {
  const kv* x = (const kv*)a;
  const kv* y = (const kv*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

typedef struct { uint32_t tile; uint32_t rank; uint32_t gid; } ent;

static int cmp_ent(const void* a, const void* b) {
  const ent* x = (const ent*)a;
  const ent* y = (const ent*)b;
  if (x->tile != y->tile) return x->tile < y->tile ? -1 : 1;
  return x->rank < y->rank ? -1 : (x->rank > y->rank);
}

/* Entries sorted by (tile, depth, index) - np.lexsort((rows, depths[rows],
 * tiles)) of frontend.py:169 with rows = ascending cloud index; ranges as
 * np.searchsorted (:171-173).  order[] receives the (depth, index) order of
 * the active Gaussians.  Returns E, or -1 if it exceeds cap. */
int64_t xgo_bin(int64_t n, int32_t width, int32_t height, const uint64_t* depth_key,
                const int32_t* n_tiles, const int32_t* rect, uint32_t* order, uint32_t* entry_splat,
                int64_t cap, int64_t* tile_ranges) {
  const int ntx = (width + TILE - 1) / TILE, nty = (height + TILE - 1) / TILE;
  const int T = ntx * nty;
  kv* a = (kv*)malloc(sizeof(kv) * (size_t)(n > 0 ? n : 1));
  int64_t na = 0, E = 0;
  for (int64_t i = 0; i < n; ++i)
    if (n_tiles[i] > 0) {
      a[na].key = depth_key[i];
      a[na].idx = (uint32_t)i;
      ++na;
      E += n_tiles[i];
    }
  qsort(a, (size_t)na, sizeof(kv), cmp_kv);
  for (int64_t s = 0; s < na; ++s) order[s] = a[s].idx;
  if (E > cap) { free(a); return -1; }
  ent* e = (ent*)malloc(sizeof(ent) * (size_t)(E > 0 ? E : 1));
  int64_t o = 0;
  for (int64_t s = 0; s < na; ++s) {
    const int32_t* r = rect + 4 * (int64_t)a[s].idx;
    for (int ty = r[1]; ty <= r[3]; ++ty)
      for (int tx = r[0]; tx <= r[2]; ++tx) {
        e[o].tile = (uint32_t)(ty * ntx + tx);
        e[o].rank = (uint32_t)s;
        e[o].gid = a[s].idx;
        ++o;
      }
  }
  qsort(e, (size_t)E, sizeof(ent), cmp_ent);
  int64_t k = 0;
  for (int t = 0; t < T; ++t) {
    tile_ranges[2 * t] = k;
    while (k < E && e[k].tile == (uint32_t)t) ++k;
    tile_ranges[2 * t + 1] = k;
  }
  for (int64_t j = 0; j < E; ++j) entry_splat[j] = e[j].gid;
  free(e);
  free(a);
  return E;
}

/* ------------------------------------------------------------------------ */
/* One float32 blend step in the engine's operation order; returns 1 if the
 * entry was blended. */
typedef struct {
  float mxr, myr, A, B, C, alpha, it;
} orec;

static orec make_rec(const double* mean2d, const float* coef, const float* inten, uint32_t g, int x0,
                     int y0) {
  orec r;
  r.mxr = (float)(mean2d[2 * g] - (double)x0);
  r.myr = (float)(mean2d[2 * g + 1] - (double)y0);
  r.A = coef[4 * g];
  r.B = coef[4 * g + 1];
  r.C = coef[4 * g + 2];
  r.alpha = coef[4 * g + 3];
  r.it = inten[g];
  return r;
}

static const float CUT2_F = (float)(POWER_CUTOFF * LOG2E);

/* p2 = A dx^2 + B dx dy + C dy^2 on the log2 scale (power * log2 e). */
static float pixel_p2(const orec* r, float fx, float fy, float* dxo, float* dyo) {
  float dx = fx - r->mxr;
  float dy = fy - r->myr;
  float adx2 = (r->A * dx) * dx;
  float bdx = r->B * dx;
  *dxo = dx;
  *dyo = dy;
  return fmaf(fmaf(r->C, dy, bdx), dy, adx2);
}

typedef struct {
  int32_t h, w;
  const double* mean2d;
  const float* coef;
  const float* inten;
  const uint32_t* entry_splat;
  const int64_t* tile_ranges;
  float* image;
  float* t_final;
  int32_t* n_contrib;
  int32_t* n_traversed;
  uint8_t* ambiguous;
  double amb_rel;
  int n_tiles;
  _Atomic int next;
} fwd_job;

static void fwd_tile(const fwd_job* j, int t) {
  const int ntx = (j->w + TILE - 1) / TILE;
  const int32_t h = j->h, w = j->w;
  const int x0 = TILE * (t % ntx), y0 = TILE * (t / ntx);
  const int64_t start = j->tile_ranges[2 * t], end = j->tile_ranges[2 * t + 1];
  for (int py = y0; py < y0 + TILE && py < h; ++py)
    for (int px = x0; px < x0 + TILE && px < w; ++px) {
      const float fx = (float)(px - x0), fy = (float)(py - y0);
      float T = 1.0f, acc = 0.0f;
      int last = -1;
      int64_t k = start;
      uint8_t amb = 0;
      for (; k < end; ++k) {
        if (fabs((double)T / FLOOR_F - 1.0) < j->amb_rel) amb = 1;
        if (T < FLOOR_F) break; /* _kernels.pyx:57-58 */
        orec r = make_rec(j->mean2d, j->coef, j->inten, j->entry_splat[k], x0, y0);
        float dx, dy;
        float p2 = pixel_p2(&r, fx, fy, &dx, &dy);
        if (p2 > 0.0f || p2 < CUT2_F) continue; /* :66-67 */
        float dens = (float)exp2((double)p2);
        float sg = r.alpha * dens;
        if (sg >= CLAMP_F) sg = CLAMP_F; /* :68-70 */
        float wgt = sg * T;
        acc = fmaf(r.it, wgt, acc); /* :71 */
        T = fmaf(-sg, T, T);        /* :72 */
        last = (int)(k - start);
      }
      const int64_t o = (int64_t)py * w + px;
      j->image[o] = acc;
      if (j->t_final) j->t_final[o] = T;
      if (j->n_contrib) j->n_contrib[o] = last + 1;
      if (j->n_traversed) j->n_traversed[o] = (int32_t)(k - start);
      if (j->ambiguous) j->ambiguous[o] = amb;
    }
}

static void* fwd_worker(void* arg) {
  fwd_job* j = (fwd_job*)arg;
  for (int t; (t = atomic_fetch_add(&j->next, 1)) < j->n_tiles;) fwd_tile(j, t);
  return NULL;
}

/* Forward blend, _kernels.pyx:41-73 per pixel.  Tiles write disjoint pixels,
 * so they are spread over XGO_THREADS (default: all online cores) threads;
 * the result does not depend on the thread count. */
void xgo_composite_fwd(int32_t h, int32_t w, const double* mean2d, const float* coef, const float* inten,
                       const uint32_t* entry_splat, const int64_t* tile_ranges, float* image,
                       float* t_final, int32_t* n_contrib, int32_t* n_traversed, uint8_t* ambiguous,
                       double amb_rel) {
  const int ntx = (w + TILE - 1) / TILE, nty = (h + TILE - 1) / TILE;
  fwd_job j = {h, w, mean2d, coef, inten, entry_splat, tile_ranges, image, t_final, n_contrib, n_traversed,
               ambiguous, amb_rel, ntx * nty, 0};
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  const char* env = getenv("XGO_THREADS");
  if (env && atoi(env) > 0) nt = atoi(env);
  if (nt > 64) nt = 64;
  if (nt > j.n_tiles / 4) nt = j.n_tiles / 4;
  if (nt <= 1) {
    fwd_worker(&j);
    return;
  }
  pthread_t th[64];
  for (long i = 0; i < nt; ++i) pthread_create(&th[i], NULL, fwd_worker, &j);
  for (long i = 0; i < nt; ++i) pthread_join(th[i], NULL);
}

/* Gradient pass (_kernels.pyx:121-177) in float64 on the float32 forward's
 * decisions.  Outputs are indexed by cloud row (n rows), accumulated. */
static void bwd_core(int32_t h, int32_t w, const double* mean2d, const float* coef, const float* inten,
                     const uint32_t* entry_splat, const int64_t* tile_ranges, const double* dl, int t_first,
                     int t_stride, double* g_mean, double* g_conic, double* g_int, double* g_alpha) {
  const int ntx = (w + TILE - 1) / TILE, nty = (h + TILE - 1) / TILE;
  const double ln2 = 0.69314718055994530942;
  int64_t cap = 64;
  int64_t* ks = (int64_t*)malloc(sizeof(int64_t) * cap);
  double* sig = (double*)malloc(sizeof(double) * cap);
  uint8_t* clamped = (uint8_t*)malloc(cap);
  for (int t = t_first; t < ntx * nty; t += t_stride) {
    const int x0 = TILE * (t % ntx), y0 = TILE * (t / ntx);
    const int64_t start = tile_ranges[2 * t], end = tile_ranges[2 * t + 1];
    for (int py = y0; py < y0 + TILE && py < h; ++py)
      for (int px = x0; px < x0 + TILE && px < w; ++px) {
        const double g = dl[(int64_t)py * w + px];
        const float fx = (float)(px - x0), fy = (float)(py - y0);
        /* float32 forward replay: which entries blend, clamped or not */
        float T = 1.0f;
        int64_t m = 0;
        for (int64_t k = start; k < end; ++k) {
          if (T < FLOOR_F) break;
          orec r = make_rec(mean2d, coef, inten, entry_splat[k], x0, y0);
          float dx, dy;
          float p2 = pixel_p2(&r, fx, fy, &dx, &dy);
          if (p2 > 0.0f || p2 < CUT2_F) continue;
          float dens = (float)exp2((double)p2);
          float sg = r.alpha * dens;
          int cl = sg >= CLAMP_F;
          if (cl) sg = CLAMP_F;
          T = fmaf(-sg, T, T);
          if (m == cap) {
            cap *= 2;
            ks = (int64_t*)realloc(ks, sizeof(int64_t) * cap);
            sig = (double*)realloc(sig, sizeof(double) * cap);
            clamped = (uint8_t*)realloc(clamped, cap);
          }
          ks[m] = k;
          clamped[m] = (uint8_t)cl;
          sig[m] = cl ? 0.99 : (double)r.alpha * exp2((double)p2);
          ++m;
        }
        if (g == 0.0 || m == 0) continue;
        /* pass 1: total (float64) */
        double acc = 0.0, Td = 1.0;
        for (int64_t q = 0; q < m; ++q) {
          orec r = make_rec(mean2d, coef, inten, entry_splat[ks[q]], x0, y0);
          acc += (double)r.it * sig[q] * Td;
          Td *= 1.0 - sig[q];
        }
        /* pass 2: reference suffix formula */
        double prefix = 0.0;
        Td = 1.0;
        for (int64_t q = 0; q < m; ++q) {
          const uint32_t j = entry_splat[ks[q]];
          orec r = make_rec(mean2d, coef, inten, j, x0, y0);
          float dxf, dyf;
          float p2 = pixel_p2(&r, fx, fy, &dxf, &dyf);
          const double dx = dxf, dy = dyf;
          const double s = sig[q];
          const double weight = s * Td;
          const double contrib = (double)r.it * weight;
          g_int[j] += g * weight;
          if (!clamped[q]) {
            const double dens = exp2((double)p2);
            const double suffix = acc - prefix - contrib;
            const double d_sigma = g * ((double)r.it * Td - suffix / (1.0 - s));
            const double a = (double)r.A / (-0.5 * LOG2E), b = (double)r.B / (-LOG2E),
                         c = (double)r.C / (-0.5 * LOG2E);
            g_alpha[j] += d_sigma * dens;
            const double gp = d_sigma * (double)r.alpha * dens;
            g_mean[2 * j] += gp * (a * dx + b * dy);
            g_mean[2 * j + 1] += gp * (b * dx + c * dy);
            g_conic[3 * j] -= 0.5 * gp * dx * dx;
            g_conic[3 * j + 1] -= gp * dx * dy;
            g_conic[3 * j + 2] -= 0.5 * gp * dy * dy;
          }
          prefix += contrib;
          Td *= 1.0 - s;
        }
      }
  }
  (void)ln2;
  free(ks);
  free(sig);
  free(clamped);
}

void xgo_composite_bwd(int32_t h, int32_t w, const double* mean2d, const float* coef, const float* inten,
                       const uint32_t* entry_splat, const int64_t* tile_ranges, const double* dl,
                       double* g_mean, double* g_conic, double* g_int, double* g_alpha) {
  bwd_core(h, w, mean2d, coef, inten, entry_splat, tile_ranges, dl, 0, 1, g_mean, g_conic, g_int, g_alpha);
}

typedef struct {
  int32_t h, w;
  const double* mean2d;
  const float* coef;
  const float* inten;
  const uint32_t* entry_splat;
  const int64_t* tile_ranges;
  const double* dl;
  int tid, nt;
  double* buf; /* [n][7]: g_mean 2, g_conic 3, g_int, g_alpha */
  int64_t n;
} bwd_job;

static void* bwd_worker(void* arg) {
  bwd_job* j = (bwd_job*)arg;
  double* b = j->buf;
  bwd_core(j->h, j->w, j->mean2d, j->coef, j->inten, j->entry_splat, j->tile_ranges, j->dl, j->tid, j->nt, b,
           b + 2 * j->n, b + 5 * j->n, b + 6 * j->n);
  return NULL;
}

/* The same gradient pass over XGO_THREADS threads (default: online cores):
 * static tile assignment, per-thread float64 accumulators summed in thread
 * order afterwards - deterministic for a given thread count, and equal to the
 * serial pass up to float64 summation order. */
void xgo_composite_bwd_mt(int32_t h, int32_t w, int64_t n, const double* mean2d, const float* coef,
                          const float* inten, const uint32_t* entry_splat, const int64_t* tile_ranges,
                          const double* dl, double* g_mean, double* g_conic, double* g_int, double* g_alpha) {
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  const char* env = getenv("XGO_THREADS");
  if (env && atoi(env) > 0) nt = atoi(env);
  if (nt > 64) nt = 64;
  const int n_tiles = ((w + TILE - 1) / TILE) * ((h + TILE - 1) / TILE);
  if (nt > n_tiles) nt = n_tiles;
  if (nt <= 1 || n <= 0) {
    xgo_composite_bwd(h, w, mean2d, coef, inten, entry_splat, tile_ranges, dl, g_mean, g_conic, g_int, g_alpha);
    return;
  }
  bwd_job jobs[64];
  pthread_t th[64];
  for (long i = 0; i < nt; ++i) {
    bwd_job jb = {h, w, mean2d, coef, inten, entry_splat, tile_ranges, dl, (int)i, (int)nt,
                  (double*)calloc((size_t)n * 7, sizeof(double)), n};
    jobs[i] = jb;
    pthread_create(&th[i], NULL, bwd_worker, &jobs[i]);
  }
  for (long i = 0; i < nt; ++i) pthread_join(th[i], NULL);
  for (long i = 0; i < nt; ++i) {
    const double* b = jobs[i].buf;
    for (int64_t r = 0; r < 2 * n; ++r) g_mean[r] += b[r];
    for (int64_t r = 0; r < 3 * n; ++r) g_conic[r] += b[2 * n + r];
    for (int64_t r = 0; r < n; ++r) g_int[r] += b[5 * n + r];
    for (int64_t r = 0; r < n; ++r) g_alpha[r] += b[6 * n + r];
    free(jobs[i].buf);
  }
}
