// Cone-beam ray-march projector of a voxel phantom: the training-target
// generator (reference pkg/src/xsplat/phantom.py:181-250, project_phantom).
//
// Per detector pixel one ray from the source through the pixel centre
// (u = x - W/2, v = y - H/2, camera direction (u/f, v/f, 1) rotated to world
// as d_cam @ R, normalised), clipped to the volume box [-extent/2,
// extent/2] by slab intersection, sampled at the midpoints of n_steps equal
// sub-steps (n_steps = ceil(max_span / step) over the whole view, step =
// step_factor * min voxel edge), each sample a trilinear interpolation of
// the densities with scipy map_coordinates(order=1, mode='constant')
// semantics (a coordinate outside [0, M-1] on any axis samples 0), the sum
// times the ray's sub-step.
//
// Numerics: float64, compiled with -fmad=false, and every per-ray / per-
// sample coordinate is computed with the reference's numpy operation order
// (dirs, slab t's, t = t_near + dt (k + 0.5), p = s + d t, idx = (p + half) /
// voxel - 0.5), so sample positions - and with them the in/out decisions -
// are bit-identical to the reference; only the interpolation weights' and
// the per-ray sum's rounding order differ (~1e-15 relative).
//
// B200 mapping: kernel 1, one thread per ray, computes the ray (direction,
// t_near, span) into the workspace and the view's maximum span (atomicMax on
// the IEEE bits of the non-negative span); kernel 2, one thread per ray,
// marches it - consecutive threads are adjacent pixels, so a warp's samples
// walk neighbouring voxels of the L2-resident volume together.
#include <math.h>

#include "xg_internal.cuh"

namespace xg {
namespace {

struct RayWs {
  double* ray;                 // [H*W][5]: dx, dy, dz, t_near, span
  unsigned long long* maxspan; // bits of the view's max span
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

size_t ray_ws(int32_t h, int32_t w, char* base, RayWs* out) {
  const size_t n = (size_t)h * (size_t)w;
  size_t off = 0;
  RayWs r;
  r.ray = (double*)(base ? base + off : nullptr);
  off += al(5 * sizeof(double) * n);
  r.maxspan = (unsigned long long*)(base ? base + off : nullptr);
  off += al(sizeof(unsigned long long));
  if (out) *out = r;
  return off + 256;
}

__global__ void k_rays(xg_volume vol, xg_cone_view v, RayWs ws) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = v.width * v.height;
  if (i >= n) return;
  const int x = i % v.width, y = i / v.width;
  // camera-frame direction (phantom.py:207-213), rotated: d = d_cam @ R
  const double u = (double)x - (double)v.width / 2.0, vv = (double)y - (double)v.height / 2.0;
  const double c0 = u / v.focal, c1 = vv / v.focal, c2 = 1.0;
  const double* R = v.rot;
  double d[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) d[j] = (c0 * R[j] + c1 * R[3 + j]) + c2 * R[6 + j];
  const double nrm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j) d[j] = d[j] / nrm;
  // slab intersection with [-extent/2, extent/2] (:216-223)
  double tn = -INFINITY, tf = INFINITY;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double half = (double)vol.m[j] * vol.voxel_size[j] / 2.0;
    const double inv = 1.0 / d[j];
    const double tlo = (-half - v.source[j]) * inv, thi = (half - v.source[j]) * inv;
    tn = fmax(tn, fmin(tlo, thi));
    tf = fmin(tf, fmax(tlo, thi));
  }
  tn = fmax(tn, 0.0);
  const double span = fmax(tf - tn, 0.0);
  double* r = ws.ray + 5 * (size_t)i;
  r[0] = d[0];
  r[1] = d[1];
  r[2] = d[2];
  r[3] = tn;
  r[4] = span;
  atomicMax(ws.maxspan, (unsigned long long)__double_as_longlong(span));
}

// One trilinear sample, map_coordinates(order=1, mode='constant', cval=0).
__device__ __forceinline__ double sample(const double* __restrict__ dens, int m0, int m1, int m2, double a,
                                         double b, double c) {
  if (!(a >= 0.0 && a <= (double)(m0 - 1) && b >= 0.0 && b <= (double)(m1 - 1) && c >= 0.0 &&
        c <= (double)(m2 - 1)))
    return 0.0;
  const int i0 = (int)a, j0 = (int)b, k0 = (int)c;  // floor (non-negative)
  const int i1 = min(i0 + 1, m0 - 1), j1 = min(j0 + 1, m1 - 1), k1 = min(k0 + 1, m2 - 1);
  const double fa = a - (double)i0, fb = b - (double)j0, fc = c - (double)k0;
  const double ga = 1.0 - fa, gb = 1.0 - fb, gc = 1.0 - fc;
  const size_t s0 = (size_t)m1 * m2;
  const double* p00 = dens + (size_t)i0 * s0 + (size_t)j0 * m2;
  const double* p01 = dens + (size_t)i0 * s0 + (size_t)j1 * m2;
  const double* p10 = dens + (size_t)i1 * s0 + (size_t)j0 * m2;
  const double* p11 = dens + (size_t)i1 * s0 + (size_t)j1 * m2;
  const double v00 = gc * __ldg(p00 + k0) + fc * __ldg(p00 + k1);
  const double v01 = gc * __ldg(p01 + k0) + fc * __ldg(p01 + k1);
  const double v10 = gc * __ldg(p10 + k0) + fc * __ldg(p10 + k1);
  const double v11 = gc * __ldg(p11 + k0) + fc * __ldg(p11 + k1);
  return ga * (gb * v00 + fb * v01) + fa * (gb * v10 + fb * v11);
}

__global__ void k_march(xg_volume vol, xg_cone_view v, RayWs ws, double step, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = v.width * v.height;
  if (i >= n) return;
  const double maxspan = __longlong_as_double((long long)*ws.maxspan);
  const double ns = ceil(maxspan / step);
  const long long n_steps = ns < 1.0 ? 1 : (long long)ns;
  const double* r = ws.ray + 5 * (size_t)i;
  const double d0 = r[0], d1 = r[1], d2 = r[2], tn = r[3], span = r[4];
  const double dt = span / (double)n_steps;
  double h[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) h[j] = (double)vol.m[j] * vol.voxel_size[j] / 2.0;
  double acc = 0.0;
  for (long long k = 0; k < n_steps; ++k) {
    const double t = tn + dt * ((double)k + 0.5);
    const double a = ((v.source[0] + d0 * t) + h[0]) / vol.voxel_size[0] - 0.5;
    const double b = ((v.source[1] + d1 * t) + h[1]) / vol.voxel_size[1] - 0.5;
    const double c = ((v.source[2] + d2 * t) + h[2]) / vol.voxel_size[2] - 0.5;
    acc += sample(vol.densities, vol.m[0], vol.m[1], vol.m[2], a, b, c);
  }
  out[i] = acc * dt;
}

}  // namespace
}  // namespace xg

using namespace xg;

extern "C" {

size_t xg_project_workspace_bytes(int32_t h, int32_t w) {
  if (h < 1 || w < 1) return 256;
  return ray_ws(h, w, nullptr, nullptr);
}

xg_status xg_project_volume(const xg_volume* vol, const xg_cone_view* view, double step_factor, double* out,
                            void* workspace, size_t workspace_bytes, void* stream) {
  if (!vol || !view || !out || !workspace || !vol->densities || view->width < 1 || view->height < 1 ||
      vol->m[0] < 1 || vol->m[1] < 1 || vol->m[2] < 1 || !(view->focal > 0.0) ||
      !(step_factor > 0.0 && step_factor <= 0.5)) {
    set_error_msg("xg_project_volume: invalid argument");
    return XG_ERR_INVALID;
  }
  if (workspace_bytes < xg_project_workspace_bytes(view->height, view->width)) {
    set_error_msg("xg_project_volume: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  RayWs ws;
  ray_ws(view->height, view->width, (char*)workspace, &ws);
  cudaMemsetAsync(ws.maxspan, 0, sizeof(unsigned long long), s);
  const double vmin = fmin(vol->voxel_size[0], fmin(vol->voxel_size[1], vol->voxel_size[2]));
  const int n = view->width * view->height;
  k_rays<<<div_up(n, 256), 256, 0, s>>>(*vol, *view, ws);
  xg_status st = check_launch("k_rays");
  if (st != XG_OK) return st;
  k_march<<<div_up(n, 128), 128, 0, s>>>(*vol, *view, ws, step_factor * vmin, out);
  return check_launch("k_march");
}

}  // extern "C"
