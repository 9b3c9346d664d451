// K3 / K4a: per-tile front-to-back compositing and its reverse replay.
//
// Reference semantics (rasterizer/_kernels.pyx:41-73, 121-177):
//   per pixel, entries of its tile in (depth, index) order; stop once
//   T < 1e-4 (tested BEFORE each entry); skip an entry if power > 0 or
//   power < -30; sigma = min(alpha e^power, 0.99); acc += i sigma T;
//   T *= 1 - sigma.  The pixel centre is the integer lattice point.
//
// B200 mapping (warp-centric).  Tracking launches (render, training): the
// unit of work is one 8x8 quarter of a 16x16 tile, owned by ONE warp (2
// vertically adjacent pixels per lane, sharing dx and the dx-only terms).
// Image-only launches (sweeps): one warp per tile, 8 rows of one column per
// lane, each 16x8 half walking its own culled entry list (compact_fwd_split).
// Units are dispatched heaviest tile first, so the load balances at
// sub-tile granularity and no warp ever waits for a sibling.  Batches are
// blended speculatively without per-pair tests and re-run exactly only where
// a pixel crosses the transmittance floor (see composite_unit).
// A warp walks its tile's entry list 32 at a time: each lane gathers one
// entry's 36 B splat record (mean re-based to the tile origin in float64,
// so dx/dy keep ~1e-6 px precision), tests it against the warp's 8x8
// sub-block with an exact ellipse/rectangle bound (max of the concave
// log-density over the rectangle vs the -30 cut-off, with margin), and the
// survivors are ballot-compacted into the warp's shared-memory slice; the
// next batch's gathers are issued before the current batch is blended.
// Culling never changes results: a culled entry has power < -30 on every
// pixel of the sub-block, which the reference skips too.
//
// Power is evaluated on the log2 scale, p2 = A2 dx^2 + B2 dx dy + C2 dy^2
// (= power * log2 e) with one MUFU.EX2 per pair (image-only: 5 per 8 rows via
// the row recurrence, blend_splat_spec_rec); the transmittance update
// T <- T - sigma T is a single fused multiply-add.
#include <stdlib.h>

#include <atomic>

#include "xg_internal.cuh"
#include "xg_sort.cuh"

namespace xg {
namespace {

#ifndef XG_COMPOSITE_WARPS
#define XG_COMPOSITE_WARPS 4
#endif
constexpr int kWarps = XG_COMPOSITE_WARPS;  // independent warps per CTA
#ifndef XG_FWD_UNROLL
#define XG_FWD_UNROLL 4
#endif
constexpr int kFwdUnroll = XG_FWD_UNROLL;
constexpr int kThreads = 32 * kWarps;
// Replay checkpoints every kCk entries of a tile (xg_splats.replay_ckpt).
__host__ __device__ constexpr int log2_exact(int x) { return x <= 1 ? 0 : 1 + log2_exact(x >> 1); }
constexpr int kCkShift = log2_exact(XG_REPLAY_CHUNK);
constexpr int kCk = 1 << kCkShift;
static_assert(kCk == XG_REPLAY_CHUNK && kCk % 32 == 0, "checkpoints sit on 32-entry batch boundaries");
constexpr float kCullMargin = 0.05f;
// image-only split path: the multiplicative row recurrence for
// recurrence-safe batches (blend_splat_spec_rec)
#ifndef XG_FWD_RECUR
#define XG_FWD_RECUR 1
#endif
constexpr bool kFwdRecur = XG_FWD_RECUR != 0;
#ifdef XG_BWD_STATS
__device__ unsigned long long g_fwd_stats[8];  // (development aid) recurrence / direct batches, survivors,
                                               // split-path batches with {both halves, one half} alive
#endif
#ifndef XG_FWD_REC_UNROLL
#define XG_FWD_REC_UNROLL 4  // measured: 1 -0.8 %, 2, 4 +0.5 % (C3) / +1.4 % (C4)
#endif
constexpr int kRecUnroll = XG_FWD_REC_UNROLL;
// split path, direct-EX2 batches (measured: 2 vs 4 splats +0.9 % at C3, no spill)
#ifndef XG_FWD_SPLIT_UNROLL
#define XG_FWD_SPLIT_UNROLL 2
#endif
constexpr int kSplitUnroll = XG_FWD_SPLIT_UNROLL;
// kClamp can only bind when alpha >= 0.99 (dens <= 1 for p2 <= 0); below a
// safety margin for the MUFU.EX2 error the clamp logic is compiled out.
constexpr float kNoClampAlpha = 0.98999f;


__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Max of the concave p2 over the rectangle of pixel centres [xa,xb]x[ya,yb]
// (tile-relative) compared against the cut-off.  The maximiser lies on the
// edge facing the mean (or is the mean), so checking the two clamped edge
// maxima is exact.
__device__ __forceinline__ bool overlaps(float mx, float my, float A, float B, float C, float xa, float xb, float ya,
                                         float yb) {
  if (!(A < -1e-30f) || !(C < -1e-30f)) return true;  // (keeps the reciprocals below finite)
  // (the edge maximiser's location only needs to be close: a misplaced
  // point lowers the computed max by O(error^2), far inside kCullMargin, so
  // the approximate MUFU.RCP division is safe - the IEEE division's slow
  // path used to cost a fifth of the kernel's instructions)
  const float dx1 = fminf(fmaxf(mx, xa), xb) - mx;
  const float dy1 = fminf(fmaxf(-B * dx1 * rcp_approx(2.f * C), ya - my), yb - my);
  const float p1 = A * dx1 * dx1 + B * dx1 * dy1 + C * dy1 * dy1;
  const float dy2 = fminf(fmaxf(my, ya), yb) - my;
  const float dx2 = fminf(fmaxf(-B * dy2 * rcp_approx(2.f * A), xa - mx), xb - mx);
  const float p2 = A * dx2 * dx2 + B * dx2 * dy2 + C * dy2 * dy2;
  return fmaxf(p1, p2) >= kCut2 - kCullMargin;
}

// One lane's gathered entry (raw, before re-basing).
struct Raw {
  double2 m;
  float4 c;
  float it;
  uint32_t g;
  bool valid;
  ushort4 r;     // reproducible reverse replay only: the splat's tile rectangle
  uint32_t off;  //   and its first slot
};

struct Unit {
  int x0, y0;            // tile origin
  int px, py0;           // this lane's pixels (px, py0) and (px, py0 + 1)
  float fx, fy0, fy1;    // tile-relative pixel centres
  float xa, xb, ya, yb;  // the warp's 8x8 sub-block (tile-relative)
  bool in0, in1;
  long long start, end;
};

__device__ __forceinline__ Unit make_unit(int tile, int quad, int ntx, int w, int h, const long long* ranges) {
  Unit u;
  const int tx = tile % ntx, ty = tile / ntx;
  u.x0 = tx * kTile;
  u.y0 = ty * kTile;
  const int lane = threadIdx.x & 31;
  const int sx = (quad & 1) * 8, sy = (quad >> 1) * 8;
  const int lx = sx + (lane & 7), ly = sy + 2 * (lane >> 3);
  u.px = u.x0 + lx;
  u.py0 = u.y0 + ly;
  u.fx = (float)lx;
  u.fy0 = (float)ly;
  u.fy1 = (float)(ly + 1);
  u.xa = (float)sx;
  u.xb = (float)(sx + 7);
  u.ya = (float)sy;
  u.yb = (float)(sy + 7);
  u.in0 = u.px < w && u.py0 < h;
  u.in1 = u.px < w && u.py0 + 1 < h;
  u.start = ranges[2 * tile];
  u.end = ranges[2 * tile + 1];
  return u;
}

// Sub-block `sub` of a tile for a warp whose lanes own 2 kP pixels each:
// kP = 1 the 8x8 quarter above; kP = 2, 4 a 16-wide block of 4 kP rows,
// lane = column lane & 15, rows py0 + 0 .. 2 kP - 1 (py0 = 2 kP (lane >> 4)
// into the block) - the per-splat shared work (record loads, dx terms,
// the warp reduction of the replay) then serves 4 kP pixels per warp lane
// pair instead of 2.
template <int kP>
__device__ __forceinline__ Unit make_sub(int tile, int sub, int ntx, int w, int h, const long long* ranges) {
  if (kP == 1) return make_unit(tile, sub, ntx, w, h, ranges);
  constexpr int kR = 2 * kP, kRows = 2 * kR;
  Unit u;
  u.x0 = (tile % ntx) * kTile;
  u.y0 = (tile / ntx) * kTile;
  const int lane = threadIdx.x & 31;
  const int lx = lane & 15, ly = sub * kRows + (lane >> 4) * kR;
  u.px = u.x0 + lx;
  u.py0 = u.y0 + ly;
  u.fx = (float)lx;
  u.fy0 = (float)ly;
  u.fy1 = (float)(ly + 1);
  u.xa = 0.f;
  u.xb = (float)(kTile - 1);
  u.ya = (float)(sub * kRows);
  u.yb = (float)(sub * kRows + kRows - 1);
  u.in0 = u.px < w && u.py0 < h;
  u.in1 = u.px < w && u.py0 + 1 < h;
  u.start = ranges[2 * tile];
  u.end = ranges[2 * tile + 1];
  return u;
}

// Next (tile, quarter) unit for this warp.  Units are the heaviest-first
// tile order x 4 quarters.  The first wave is dealt statically: warp w of
// CTA c takes unit G*w + c (w even) or G*w + G-1-c (w odd), so every CTA -
// and with an even CTA count per SM every SM - starts with the same mix of
// heavy and light units (a shared counter would hand them out in arrival
// order).  After that, warps pull the remaining (lightest) units from the
// counter.
// order: tiles (4 units each, kUnits = false) or units (kUnits = true).
template <bool kUnits, int kSubs = 4>
__device__ __forceinline__ bool next_unit(const int* order, uint32_t* work, int n_tiles, bool& first,
                                          int& tile, int& quad) {
  const uint32_t n_units = (uint32_t)kSubs * (uint32_t)n_tiles;
  const uint32_t G = gridDim.x, w = threadIdx.x >> 5;
  const uint32_t dealt = min(n_units, G * (uint32_t)kWarps);
  uint32_t k = n_units;
  if (first) {
    first = false;
    k = G * w + ((w & 1u) ? G - 1u - blockIdx.x : blockIdx.x);
  }
  if (k >= dealt) {
    uint32_t d = 0;
    if ((threadIdx.x & 31) == 0) d = atomicAdd(work, 1u);
    k = dealt + __shfl_sync(0xffffffffu, d, 0);
  }
  if (k >= n_units) return false;
  if (kUnits) {
    const int uidx = order[k];
    tile = uidx >> 2;
    quad = uidx & 3;
  } else {
    tile = order[k / kSubs];
    quad = (int)(k % kSubs);
  }
  return true;
}

struct FwdArgs {
  const double2* mean2d;
  const float4* coef;
  const float* inten;
  const uint32_t* entry;
  const long long* ranges;
  const int* order;        // tiles, heaviest first
  uint32_t* work;          // queue head (zeroed before launch)
  int n_tiles;
  float* image;
  float* t_final;
  int* n_contrib;
  const float* target;
  double* l1_sum;
  int* unit_cost;  // optional: entries each unit's reverse replay will walk
  const uint32_t* n_entries;  // counters[XG_CTR_ENTRIES] (or null)
  long long cap;              // entry capacity: an overflowed view is skipped (re-binned by the caller)
  int ntx, w, h;
  float2* ckpt;               // optional (tracking only): (T, acc) before every kCk-th entry
  // streamed replay (xg_composite_train_pair): each finished tile publishes its
  // reverse-replay chunks to this ring, epoch-tagged, for the concurrently
  // running k_composite_bwd_stream
  unsigned long long* ring;   // [ring_cap] (tile | chunk << 20 | epoch << 40), or null
  long long ring_cap;
  uint32_t* ring_ctr;         // counters + XG_CTR_ITEMS: [0] slots reserved, [1] tiles published
  uint32_t epoch;             // 24 bits
};

// Checkpoint slot of entry kCk * m of the tile whose list starts at `start`:
// unique per (tile, m >= 1) and < entries / kCk + n_tiles + 1.
__device__ __forceinline__ long long ckpt_slot(long long start, int tile, long long m) {
  return (start >> kCkShift) + tile + m;
}

// Forward records in shared memory, signs folded so that every per-pixel
// step of the lane's two pixels is ONE packed FP32x2 instruction (sm_100
// FADD2 / FFMA2 / FMUL2, two IEEE round-to-nearest results per issue slot):
//   dy = fy + (-my)           == fy - my
//   s  = (-alpha) * 2^p2      == -sigma
//   w  = s * T                == -(sigma T)
//   acc = fma(-i, w, acc)     == fma(i, sigma T, acc)
//   T   = fma(s, T, T)        == fma(-sigma, T, T)
// - bit for bit the reference-order float32 operations the oracle performs.
struct FRec {
  float4 a;  // mx (tile-relative), -my, A2, B2
  float4 b;  // C2, -alpha, -intensity, 0
};

// The p2 <= 0 test can be dropped for a splat whose quadratic form
// M = -[[A2, B2/2], [B2/2, C2]] is positive definite with
// lambda_min / lambda_max > 2.0000001 u (u = 2^-24): the computed
// p2 = fma(fma(C2, dy, B2 dx), dy, (A2 dx) dx) differs from the exact form
// by at most 2.0000001 u lambda_max |v|^2 (five roundings), so it cannot
// round above zero.  lambda_min / lambda_max >= det / tr^2;
// the float test det >= 1e-6 tr^2 leaves a 7x margin over the rounding of
// det and tr themselves.
__device__ __forceinline__ bool well_conditioned(float A, float B, float C) {
  const float det = A * C - 0.25f * B * B;
  const float tr = A + C;
  return (A < 0.f) && (C < 0.f) && (det < INFINITY) && (det >= 1e-6f * tr * tr);
}

__device__ __forceinline__ float2 bc(float x) { return make_float2(x, x); }

// (p2 >= cut && T >= floor) ? sg : 0 as FSETP, FSETP.AND, FSEL
__device__ __forceinline__ float select_ok(float sg, float p2, float T) {
  float r;
  asm("{\n\t.reg .pred q, o;\n\t"
      "setp.ge.f32 q, %3, %5;\n\t"
      "setp.ge.and.f32 o, %2, %4, q;\n\t"
      "selp.f32 %0, %1, 0f00000000, o;\n\t}"
      : "=f"(r)
      : "f"(sg), "f"(p2), "f"(T), "f"(kCut2), "f"(kFloor));
  return r;
}

// One splat, one vertically adjacent pixel pair of the lane: the blend step
// of _kernels.pyx:57-72.  kGeneral keeps the sigma <= 0.99 clamp (only
// alpha >= 0.99 can reach it) and the p2 <= 0 test (only ill-conditioned
// splats can need it); both are warp-uniform per batch.  Records the last
// blended entry (n_contrib).
template <bool kGeneral, bool kTrack, bool kLa = false>
__device__ __forceinline__ void blend_pair(const FRec& r, int krel, float2 dy, float bdx, float adx2, float2& T,
                                           float2& acc, int& last0, int& last1) {
  const float2 p = __ffma2_rn(__ffma2_rn(bc(r.b.x), dy, bc(bdx)), dy, bc(adx2));
  // kLa (image-only split records, b.y holds the recurrence factor): sigma
  // = 2^(p2 + log2 alpha), as in the speculative image-only step
  float2 sg = kLa ? make_float2(-ex2_approx(p.x + r.b.w), -ex2_approx(p.y + r.b.w))
                  : __fmul2_rn(bc(r.b.y), make_float2(ex2_approx(p.x), ex2_approx(p.y)));
  if (kGeneral) {
    sg.x = fmaxf(sg.x, -kClamp);
    sg.y = fmaxf(sg.y, -kClamp);
  }
  bool ok0 = (p.x >= kCut2) & (T.x >= kFloor);
  bool ok1 = (p.y >= kCut2) & (T.y >= kFloor);
  if (kGeneral) {
    ok0 &= p.x <= 0.f;
    ok1 &= p.y <= 0.f;
  }
  if (kGeneral || kTrack) {
    sg.x = ok0 ? sg.x : 0.f;
    sg.y = ok1 ? sg.y : 0.f;
  } else {
    // one chained compare + one select per pixel (left to itself the
    // compiler splits the conjunction into two compare/select pairs)
    sg.x = select_ok(sg.x, p.x, T.x);
    sg.y = select_ok(sg.y, p.y, T.y);
  }
  const float2 w = __fmul2_rn(sg, T);
  acc = __ffma2_rn(bc(r.b.z), w, acc);
  T = __ffma2_rn(sg, T, T);
  if (kTrack) {
    last0 = ok0 ? krel : last0;
    last1 = ok1 ? krel : last1;
  }
}

// One splat, the lane's kP pixel pairs (one column: dx and the dx-only
// terms computed once).
template <bool kGeneral, bool kTrack, int kP, bool kLa = false>
__device__ __forceinline__ void blend_splat(const FRec& r, int krel, float fx, const float2 (&fy)[kP],
                                            float2 (&T)[kP], float2 (&acc)[kP], int (&last)[2 * kP]) {
  const float dx = __fsub_rn(fx, r.a.x);
  const float adx2 = __fmul_rn(__fmul_rn(r.a.z, dx), dx);
  const float bdx = __fmul_rn(r.a.w, dx);
#pragma unroll
  for (int i = 0; i < kP; ++i)
    blend_pair<kGeneral, kTrack, kLa>(r, krel, __fadd2_rn(fy[i], bc(r.a.y)), bdx, adx2, T[i], acc[i], last[2 * i],
                                      last[2 * i + 1]);
}

// Record half of the gather (the entry index is loaded one batch earlier).
__device__ __forceinline__ Raw fetch(uint32_t g, bool valid, const double2* __restrict__ mean2d,
                                     const float4* __restrict__ coef, const float* __restrict__ inten,
                                     const ushort4* __restrict__ rect = nullptr,
                                     const uint32_t* __restrict__ slot_off = nullptr) {
  Raw r;
  r.valid = valid;
  r.g = g;
  if (valid) {
    r.m = __ldg(mean2d + g);
    r.c = __ldg(coef + g);
    r.it = __ldg(inten + g);
    if (rect) {  // (issued with the record: the slot is ready at compaction)
      r.r = __ldg(rect + g);
      r.off = __ldg(slot_off + g);
    }
  }
  return r;
}

__device__ __forceinline__ uint32_t entry_at(const uint32_t* __restrict__ entry, long long k, long long hi) {
  return k < hi ? __ldg(entry + k) : 0u;
}

// Re-base, cull against the warp's sub-block, ballot-compact the survivors
// into the warp's shared slice.  general = some survivor needs the clamp or
// the p2 <= 0 test.
__device__ __forceinline__ int compact_fwd(const Raw& raw, int krel, const Unit& u, FRec* s_rec, int* s_k,
                                           bool& general) {
  FRec r;
  bool keep = false, gen = false;
  if (raw.valid) {
    const float mx = (float)(raw.m.x - (double)u.x0), my = (float)(raw.m.y - (double)u.y0);
    const float A = raw.c.x, B = raw.c.y, C = raw.c.z, alpha = raw.c.w;
    keep = overlaps(mx, my, A, B, C, u.xa, u.xb, u.ya, u.yb);
    gen = !(alpha < kNoClampAlpha) || !well_conditioned(A, B, C);
    r.a = make_float4(mx, -my, A, B);
    r.b = make_float4(C, -alpha, -raw.it, __log2f(alpha));
  }
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  general = __any_sync(0xffffffffu, keep && gen);
  if (keep) {
    const int pos = __popc(bal & lanemask_lt());
    s_rec[pos] = r;
    s_k[pos] = krel;
  }
  __syncwarp();
  return __popc(bal);
}

// Split-half compaction (image-only, whole-tile warps): every entry is culled
// against both 16x8 halves; half h's survivors go to s_rec[32 h ..] in entry
// order, and the shorter list is padded with null splats (A2 = B2 = C2 = 0,
// alpha = 0, log2 alpha = -inf: sigma = 0, an exact no-op in every blend
// variant) to the longer one's length, which is returned.  Lanes 0-15 then
// walk the top list, lanes 16-31 the bottom one: the cull granularity of
// 16x8 sub-blocks with the per-splat column work shared by 8 pixels a lane.
// p2 + log2 alpha at a tile-relative pixel (the recurrence-safety test)
__device__ __forceinline__ float p2_at(float mx, float my, float A, float B, float C, float la, float x, float y) {
  const float dx = x - mx, dy = y - my;
  return fmaf(fmaf(C, dy, B * dx), dy, fmaf(A * dx, dx, la));
}

template <int kP = 4, bool kTrack = false>
__device__ __forceinline__ int compact_fwd_split(const Raw& raw, const Unit& u, FRec* s_rec, bool& general,
                                                 bool& rec_safe, int krel = 0, int* s_k = nullptr) {
  // the warp's sub-block is rows [ya, yb] (16 x 4 kP); half h = rows
  // ya + 2 kP h .. ya + 2 kP h + 2 kP - 1 (lanes 16 h .. 16 h + 15)
  constexpr int kR = 2 * kP;
  FRec r;
  bool k0 = false, k1 = false, gen = false, unsafe = false;
  if (raw.valid) {
    const float mx = (float)(raw.m.x - (double)u.x0), my = (float)(raw.m.y - (double)u.y0);
    const float A = raw.c.x, B = raw.c.y, C = raw.c.z, alpha = raw.c.w;
    const float la = __log2f(alpha);
    k0 = overlaps(mx, my, A, B, C, u.xa, u.xb, u.ya, u.ya + (float)(kR - 1));
    k1 = overlaps(mx, my, A, B, C, u.xa, u.xb, u.ya + (float)kR, u.yb);
    gen = !(alpha < kNoClampAlpha) || !well_conditioned(A, B, C);
    r.a = make_float4(mx, -my, A, B);
    // image-only records carry the row recurrence's per-splat factor
    // 2^(8 C2) in b.y (one MUFU per entry here instead of one per splat and
    // lane in the blend); the exact re-run then takes sigma = 2^(p2 + la)
    r.b = make_float4(C, kTrack ? -alpha : ex2_approx(8.f * C), -raw.it, la);
    if (kFwdRecur && (k0 || k1)) {
      // the multiplicative row recurrence (blend_splat_spec_rec) of half h
      // starts from E_0 = 2^p2 at rows 8h, 8h + 1: those must be normal
      // floats (the concave p2 is smallest at a corner of that 16 x 2 strip);
      // later rows may underflow harmlessly (their true sigma is even
      // smaller).  The ratios 2^(p2(dy + 2) - p2(dy)), linear in (dx, dy),
      // and 2^(8 C2) must stay within 2^+-120.
      constexpr float e = (float)(kTile - 1), hh = (float)kR;
      const float mdx = fmaxf(fabsf(mx), fabsf(e - mx)), mdy = fmaxf(fabsf(my - u.ya), fabsf(u.yb - my));
      const float dmax = 4.f * fabsf(C) * mdy + fabsf(4.f * C) + 2.f * fabsf(B) * mdx;
      unsafe = !(dmax <= 120.f) || !(C >= -15.f);
      // A flushed E_0 (p2 + la < -126) is harmless when no row within 7 of
      // it in the lane's column is one the reference blends (p2 >= kCut2):
      // along a column p2 = C2 (y - y*)^2 + P* with P* <= 0, so a blended row
      // has |y - y*| <= a = sqrt(-kCut2 / |C2|) and p2 rises towards it by at
      // most |C2| ((a + 7)^2 - a^2) = 14 sqrt(-kCut2 |C2|) + 49 |C2|; if that
      // stays below 126 + kCut2 + la, flushed rows only drop pairs the
      // reference skips.  True for every splat wider than ~1.4 px (all
      // BASELINE clouds); narrower ones keep the corner test.
      const float aC = -C;
      const bool flush_ok = 14.f * sqrtf(-kCut2 * aC) + 49.f * aC <= (126.f + kCut2) + la - 1.f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!flush_ok && (h ? k1 : k0)) {
          const float y0 = u.ya + h * hh, y1 = y0 + 1.f;
          const float pmin = fminf(fminf(p2_at(mx, my, A, B, C, la, 0.f, y0), p2_at(mx, my, A, B, C, la, e, y0)),
                                   fminf(p2_at(mx, my, A, B, C, la, 0.f, y1), p2_at(mx, my, A, B, C, la, e, y1)));
          unsafe |= !(pmin >= -125.f);
        }
      }
    }
  }
  const unsigned b0 = __ballot_sync(0xffffffffu, k0), b1 = __ballot_sync(0xffffffffu, k1);
  general = __any_sync(0xffffffffu, (k0 || k1) && gen);
  rec_safe = kFwdRecur && !__any_sync(0xffffffffu, unsafe);
  const unsigned lt = lanemask_lt();
  if (k0) s_rec[__popc(b0 & lt)] = r;
  if (k1) s_rec[32 + __popc(b1 & lt)] = r;
  if (s_k) {  // (tracking launches: the entry index of every survivor, per half)
    if (k0) s_k[__popc(b0 & lt)] = krel;
    if (k1) s_k[32 + __popc(b1 & lt)] = krel;
  }
  const int c0 = __popc(b0), c1 = __popc(b1), n = c0 > c1 ? c0 : c1;
  const int lane = threadIdx.x & 31;
  // null splat padding the shorter half: mean 1e30 px away with A2 = -1 puts
  // p2 at -inf at every pixel, so sigma = 0 exactly in every blend variant
  // and no pixel ever records it as a blended (p2 >= cut) entry
  FRec z;
  z.a = make_float4(1e30f, 0.f, -1.f, 0.f);
  z.b = make_float4(0.f, 0.f, 0.f, -INFINITY);
  if (lane >= c0 && lane < n) s_rec[lane] = z;
  if (lane >= c1 && lane < n) s_rec[32 + lane] = z;
  __syncwarp();
  return n;
}

// Image-only speculative step (no per-pair tests; see composite_unit): the
// opacity rides in the exponent, sigma = 2^(p2 + log2 alpha) (record b.w),
// so a pair costs FADD2 dy, 2 FFMA2 p2, 2 MUFU.EX2, FMUL2 sigma T, FFMA2 acc,
// FFMA2 T.  Only batches of well-conditioned splats with alpha < 0.98999
// take it (p2 <= 0 exactly, sigma <= 0.99 without the clamp).  Entries the
// reference skips for power < -30 are blended here with sigma < 9.4e-14:
// T * (1 - sigma) rounds back to T exactly, acc moves by < 1e-13 i T.
template <int kP>
__device__ __forceinline__ void blend_splat_spec(const FRec& r, float fx, const float2 (&fy)[kP], float2 (&T)[kP],
                                                 float2 (&acc)[kP]) {
  const float dx = __fsub_rn(fx, r.a.x);
  const float adx2 = __fmaf_rn(__fmul_rn(r.a.z, dx), dx, r.b.w);
  const float bdx = __fmul_rn(r.a.w, dx);
  const float ni = -r.b.z;  // +intensity (folded into FFMA2's negate)
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    const float2 dy = __fadd2_rn(fy[i], bc(r.a.y));
    const float2 p = __ffma2_rn(__ffma2_rn(bc(r.b.x), dy, bc(bdx)), dy, bc(adx2));
    const float2 e = make_float2(ex2_approx(p.x), ex2_approx(p.y));
    const float2 w = __fmul2_rn(e, T[i]);
    acc[i] = __ffma2_rn(bc(ni), w, acc[i]);
    T[i] = __ffma2_rn(make_float2(-e.x, -e.y), T[i], T[i]);
  }
}

// Speculative step with the multiplicative row recurrence (split-half
// whole-tile warps, 4 pixel pairs per lane, rows dy0 + 0 .. 7): along a
// column, p2(dy + 2) - p2(dy) = 4 C2 dy + 4 C2 + 2 B2 dx is linear in dy, so
//   E_{i+1} = E_i * S_i,  S_{i+1} = S_i * 2^(8 C2)
// with E_0 = 2^p2 of rows 0, 1 and S_0 = 2^(p2(dy0 + 2) - p2(dy0)) of rows
// 0, 1: 5 MUFU.EX2 per splat and lane instead of 8 (the kernel is EX2-bound).
// Every factor stays within 2^+-120 (the compaction's rec_safe test);
// relative error a few ulp after the 3 products.
template <int kP = 4>
__device__ __forceinline__ void blend_splat_spec_rec(const FRec& r, float fx, const float2 (&fy)[kP], float2 (&T)[kP],
                                                     float2 (&acc)[kP]) {
  const float dx = __fsub_rn(fx, r.a.x);
  const float adx2 = __fmaf_rn(__fmul_rn(r.a.z, dx), dx, r.b.w);
  const float bdx = __fmul_rn(r.a.w, dx);
  const float C = r.b.x, ni = -r.b.z;
  const float c4 = 4.f * C;
  const float q4 = r.b.y;  // 2^(8 C2), from the compaction (compact_fwd_split, image-only)
  const float2 dy0 = __fadd2_rn(fy[0], bc(r.a.y));
  const float2 p0 = __ffma2_rn(__ffma2_rn(bc(C), dy0, bc(bdx)), dy0, bc(adx2));
  const float2 d0 = __ffma2_rn(bc(c4), dy0, bc(__fmaf_rn(2.f, bdx, c4)));
  float2 E = make_float2(ex2_approx(p0.x), ex2_approx(p0.y));
  float2 S = make_float2(ex2_approx(d0.x), ex2_approx(d0.y));
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    if (i > 0) {
      E = __fmul2_rn(E, S);
      S = __fmul2_rn(S, bc(q4));
    }
    const float2 w = __fmul2_rn(E, T[i]);
    acc[i] = __ffma2_rn(bc(ni), w, acc[i]);
    T[i] = __ffma2_rn(make_float2(-E.x, -E.y), T[i], T[i]);
  }
}

template <int kP, int kU = kFwdUnroll>
__device__ __forceinline__ void blend_batch_spec(const FRec* rec, int cnt, float fx, const float2 (&fy)[kP],
                                                 float2 (&T)[kP], float2 (&acc)[kP]) {
#pragma unroll kU
  for (int q = 0; q < cnt; ++q) blend_splat_spec<kP>(rec[q], fx, fy, T, acc);
}

// Tracking speculative step (training forward): sigma = alpha 2^p2 as in
// the exact path, so T (and t_final, the checkpoints) stay bit-identical to
// it - a pair below the cut-off has sigma < 9.4e-14 and T - sigma T rounds
// to T; only acc moves, by < 1e-13 i T.  The last blended entry (n_contrib)
// is exact: live pixels (T >= floor over the whole batch, else the batch is
// re-run) record every entry with p2 >= cut.
template <int kP>
__device__ __forceinline__ void blend_splat_spec_track(const FRec& r, int krel, float fx, const float2 (&fy)[kP],
                                                       const bool (&live)[2 * kP], float2 (&T)[kP],
                                                       float2 (&acc)[kP], int (&last)[2 * kP]) {
  const float dx = __fsub_rn(fx, r.a.x);
  const float adx2 = __fmul_rn(__fmul_rn(r.a.z, dx), dx);
  const float bdx = __fmul_rn(r.a.w, dx);
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    const float2 dy = __fadd2_rn(fy[i], bc(r.a.y));
    const float2 p = __ffma2_rn(__ffma2_rn(bc(r.b.x), dy, bc(bdx)), dy, bc(adx2));
    const float2 sg = __fmul2_rn(bc(r.b.y), make_float2(ex2_approx(p.x), ex2_approx(p.y)));
    const float2 w = __fmul2_rn(sg, T[i]);
    acc[i] = __ffma2_rn(bc(r.b.z), w, acc[i]);
    T[i] = __ffma2_rn(sg, T[i], T[i]);
    last[2 * i] = (live[2 * i] && p.x >= kCut2) ? krel : last[2 * i];
    last[2 * i + 1] = (live[2 * i + 1] && p.y >= kCut2) ? krel : last[2 * i + 1];
  }
}

template <bool kGeneral, bool kTrack, int kP, bool kLa = false>
__device__ __forceinline__ void blend_batch(const FRec* rec, const int* kk, int cnt, float fx, const float2 (&fy)[kP],
                                            float2 (&T)[kP], float2 (&acc)[kP], int (&last)[2 * kP]) {
  constexpr int kU = (!kTrack && kP == 4) ? kSplitUnroll : kFwdUnroll;  // (split image-only kernels: fewer registers)
#pragma unroll kU
  for (int q = 0; q < cnt; ++q)
    blend_splat<kGeneral, kTrack, kP, kLa>(rec[q], kTrack ? kk[q] : 0, fx, fy, T, acc, last);
}

// 5 CTAs (20 warps) per SM: ptxas fits the image-only variant in 96
// registers; measured 5 % faster than the unbounded 97-register build
#ifndef XG_FWD_MIN_CTAS
#define XG_FWD_MIN_CTAS 5
#endif
// pixel pairs per lane (make_sub): image-only launches / tracking launches
#ifndef XG_FWD_PAIRS
#define XG_FWD_PAIRS 4  // whole-tile warps with split-half entry lists (XG_FWD_SPLIT); measured before the
                        // split: 1 -> 2 pairs +5 % fps, 4 pairs (one 16x16 cull) -6 %
#endif
#ifndef XG_FWD_TRACK_PAIRS
#define XG_FWD_TRACK_PAIRS 1  // (C2 training: quarter tiles balance better; 2 pairs +5 % per iteration)
#endif
#ifndef XG_FWD_MIN_CTAS_WIDE
#define XG_FWD_MIN_CTAS_WIDE 4
#endif
#ifndef XG_FWD_LITE_PAIRS
#define XG_FWD_LITE_PAIRS 1  // the trainer's forward: quarter tiles.  2 = 16 x 8 half tiles with split 16 x 4
                             // lists (the image-only kernel's scheme): measured +9 % per C2 iteration (round 2)
#endif
constexpr int kFwdPairs = XG_FWD_PAIRS, kFwdTrackPairs = XG_FWD_TRACK_PAIRS, kFwdLitePairs = XG_FWD_LITE_PAIRS;
// image-only launches: speculative test-free batches (blend_batch_spec)
#ifndef XG_FWD_SPEC
#define XG_FWD_SPEC 1
#endif
constexpr bool kSpec = XG_FWD_SPEC != 0;
// tracking launches (training forward): speculative batches with exact
// n_contrib / t_final (blend_splat_spec_track)
#ifndef XG_FWD_SPEC_TRACK
#define XG_FWD_SPEC_TRACK 1
#endif
constexpr bool kSpecTrack = XG_FWD_SPEC_TRACK != 0;
// image-only launches: one warp per 16x16 tile (4 pixel pairs per lane),
// each 16x8 half with its own culled entry list (compact_fwd_split)
#ifndef XG_FWD_SPLIT
#define XG_FWD_SPLIT 1  // vs 16x8 sub-block warps: C3 within noise (+0.3 %), C4 +3.5 %
#endif
constexpr bool kFwdSplit = XG_FWD_SPLIT != 0;
static_assert(!kFwdSplit || kFwdPairs == 4, "split-half units cover whole tiles (XG_FWD_PAIRS=4)");
// split path: two 32-record lists + the batch-start (T, acc) of the lane's
// 8 pixels kept in shared memory for a re-run (frees 16 registers)
constexpr int kRecPerWarp = kFwdSplit ? 128 : 32;
static_assert((kFwdPairs == 1 || kFwdPairs == 2 || kFwdPairs == 4) &&
                  (kFwdTrackPairs == 1 || kFwdTrackPairs == 2 || kFwdTrackPairs == 4) && kWarps % 4 == 0,
              "sub-blocks of 4, 8 or 16 rows; CTAs of whole tiles");
template <bool kTrack, bool kLite = false>
__host__ __device__ constexpr int fwd_pairs() { return kTrack ? (kLite ? kFwdLitePairs : kFwdTrackPairs) : kFwdPairs; }
__host__ __device__ constexpr int min_ctas(int kP) { return kP == 1 ? XG_FWD_MIN_CTAS : XG_FWD_MIN_CTAS_WIDE; }

// TMA A/B (XG_FWD_TMA=1, image-only split path): the tile's entry-index
// list is streamed into shared memory by cp.async.bulk in 256-entry chunks
// (double-buffered per warp, mbarrier completion), replacing the warp's
// coalesced LDG of 32 indices per batch; the splat records stay register
// gathers (LDG).  Measured: no gain - the default stays LDG.
#ifndef XG_FWD_TMA
#define XG_FWD_TMA 0
#endif
constexpr int kTmaChunkShift = 8, kTmaChunk = 1 << kTmaChunkShift;
struct __align__(16) TmaBuf {
  unsigned long long mbar[2];
  uint32_t idx[2][kTmaChunk + 4];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_issue(TmaBuf* tb, const uint32_t* __restrict__ entry, long long base,
                                          long long end, int c) {
  const long long lo = base + ((long long)c << kTmaChunkShift);
  const long long n = min((long long)kTmaChunk, end - lo);
  const uint32_t bytes = (uint32_t)((n * 4 + 15) & ~15ll);  // 16 B multiple (the buffers carry 4 slack entries)
  const uint32_t mb = smem_u32(&tb->mbar[c & 1]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (generic reads of the buffer precede the rewrite)
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(tb->idx[c & 1])), "l"(entry + lo), "r"(bytes), "r"(mb) : "memory");
}

__device__ __forceinline__ void tma_wait(TmaBuf* tb, int c) {
  const uint32_t mb = smem_u32(&tb->mbar[c & 1]), parity = (uint32_t)((c >> 1) & 1);
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(mb), "r"(parity) : "memory");
}

// One sub-block unit of the forward: the warp walks the tile's entry list
// and writes the sub-block's pixels.
// kLite (training forward, tracking): speculative batches use the
// image-only step (no per-pair contributor tracking); a pixel that terminates
// gets its exact last blended entry from the re-run of the crossing batch, a
// pixel still above the floor at the end of its list gets the list's last
// entry - the reverse replay's start (entries past the true last have
// power < -30, exact no-ops up to < 1e-13 there).
template <bool kTrack, int kP, bool kLite = false>
__device__ __forceinline__ void composite_unit(const FwdArgs& a, int tile, int sub, FRec* rec, int* kk,
                                               TmaBuf* tb = nullptr) {
  constexpr int kR = 2 * kP;
  // split-half entry lists: image-only whole-tile warps (kP = 4) and the
  // trainer's tracking forward on 16 x 8 half tiles (kP = 2, kLite)
  constexpr bool kSplitPath = kSpec && kFwdSplit && (kTrack ? (kLite && kSpecTrack && kP == 2) : kP == 4);
  const int lane = threadIdx.x & 31;
  FRec* const rh = kSplitPath ? rec + 32 * (lane >> 4) : rec;  // this lane's (half's) entry list
  int* const kh = kSplitPath ? kk + 32 * (lane >> 4) : kk;      //   and its entry indices (tracking)
  const Unit u = make_sub<kP>(tile, sub, a.ntx, a.w, a.h, a.ranges);
  float2 fy[kP], T[kP], acc[kP], Tf[kP];  // Tf: final T of a pixel parked at T = 0 (tracking + speculation)
  int last[kR];
  bool any_in = false;
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    fy[i] = make_float2(u.fy0 + (float)(2 * i), u.fy0 + (float)(2 * i + 1));
    const bool in0 = u.px < a.w && u.py0 + 2 * i < a.h, in1 = u.px < a.w && u.py0 + 2 * i + 1 < a.h;
    T[i] = make_float2(in0 ? 1.f : 0.f, in1 ? 1.f : 0.f);
    acc[i] = make_float2(0.f, 0.f);
    Tf[i] = make_float2(0.f, 0.f);
    last[2 * i] = last[2 * i + 1] = -1;
    any_in |= in0 | in1;
  }
  bool alive = __any_sync(0xffffffffu, any_in);
  // TMA variant: index chunks [base + 256 c, base + 256 (c + 1)) in buffer c & 1
  constexpr bool kTma = XG_FWD_TMA && kSplitPath;
  const long long tbase = u.start & ~3ll;  // 16 B aligned
  int tma_issued = 0, tma_ready = -1;
  const int tma_chunks = kTma ? (int)((u.end - tbase + kTmaChunk - 1) >> kTmaChunkShift) : 0;
  if (kTma && tma_chunks > 0) {
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tb->mbar[0])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tb->mbar[1])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      tma_issue(tb, a.entry, tbase, u.end, 0);
      if (tma_chunks > 1) tma_issue(tb, a.entry, tbase, u.end, 1);
    }
    tma_issued = tma_chunks > 1 ? 2 : 1;
    __syncwarp();
  }
  // index k of the tile list (k < end), from shared memory (TMA) or global
  auto idx_at = [&](long long k) -> uint32_t {
    if (!kTma) return entry_at(a.entry, k, u.end);
    if (k >= u.end) return 0u;
    const int c = (int)((k - tbase) >> kTmaChunkShift);
    return tb->idx[c & 1][(k - tbase) & (kTmaChunk - 1)];
  };
  auto tma_need = [&](long long kmax) {  // chunks up to kmax's have landed (warp-uniform)
    if (!kTma) return;
    kmax = min(kmax, u.end - 1);
    const int c = (int)((kmax - tbase) >> kTmaChunkShift);
    while (tma_ready < c) tma_wait(tb, ++tma_ready);
  };
  // two-stage prefetch: entry indices one batch ahead of the records
  tma_need(u.start + 63);
  Raw nxt = fetch(idx_at(u.start + lane), u.start + lane < u.end, a.mean2d, a.coef, a.inten);
  uint32_t g_nxt = idx_at(u.start + 32 + lane);
  for (long long b0 = u.start; alive && b0 < u.end; b0 += 32) {
    if (kTrack && a.ckpt) {
      // state before entry b0 for the chunked reverse replay; a warp that
      // stopped early never reaches later boundaries, but then none of its
      // pixels blends past them and the replay restarts from the final state
      const long long rel = b0 - u.start;
      if (rel > 0 && (rel & (kCk - 1)) == 0) {
        float2* c = a.ckpt + 256 * ckpt_slot(u.start, tile, rel >> kCkShift) + (u.py0 - u.y0) * kTile +
                    (u.px - u.x0);
#pragma unroll
        for (int r = 0; r < kR; ++r)
          if (u.px < a.w && u.py0 + r < a.h)
            c[r * kTile] = (r & 1) ? make_float2(T[r >> 1].y, acc[r >> 1].y) : make_float2(T[r >> 1].x, acc[r >> 1].x);
      }
    }
    const Raw cur = nxt;
    bool general;
    bool rec_safe = false;
    const int cnt = kSplitPath ? compact_fwd_split<kP, kTrack>(cur, u, rec, general, rec_safe,
                                                               (int)(b0 - u.start) + lane, kTrack ? kk : nullptr)
                               : compact_fwd(cur, (int)(b0 - u.start) + lane, u, rec, kk, general);
    nxt = fetch(g_nxt, b0 + 32 + lane < u.end, a.mean2d, a.coef, a.inten);
    if (kTma) {
      tma_need(b0 + 95);
      g_nxt = idx_at(b0 + 64 + lane);
      // a buffer is refilled (chunk c + 2) once no later read targets chunk c:
      // reads from here on are at k >= b0 + 96
      while (tma_issued < tma_chunks && tbase + ((long long)(tma_issued - 1) << kTmaChunkShift) <= b0 + 96 &&
             tma_ready >= tma_issued - 2) {
        __syncwarp();
        if (lane == 0) tma_issue(tb, a.entry, tbase, u.end, tma_issued);
        ++tma_issued;
      }
    } else {
      g_nxt = entry_at(a.entry, b0 + 64 + lane, u.end);
    }
    if (!(kTrack ? kSpecTrack : kSpec)) {
      if (general)  // warp-uniform, per batch of 32 entries
        blend_batch<true, kTrack, kP>(rec, kk, cnt, u.fx, fy, T, acc, last);
      else
        blend_batch<false, kTrack, kP>(rec, kk, cnt, u.fx, fy, T, acc, last);
    } else {
      // Speculate that no live pixel crosses the transmittance floor inside
      // the batch and blend without the per-pair T test; a terminated pixel
      // holds T = 0 (its final T kept in Tf), which makes every later step an
      // exact no-op.  If a pixel did cross, the warp restores the batch-start
      // state and re-runs the batch with the reference's tests (one extra
      // batch per crossing).
      bool redo = general;
      if (!general) {
        float2 T0[kP], A0[kP];
        int L0[kR];
        bool lv[kR];
        float4* const sv = reinterpret_cast<float4*>(rec + 64) + lane;  // (split path only)
#pragma unroll
        for (int i = 0; i < kP; ++i) {
          if (kSplitPath) {
            sv[32 * i] = make_float4(T[i].x, T[i].y, acc[i].x, acc[i].y);
          } else {
            T0[i] = T[i];
            A0[i] = acc[i];
          }
          lv[2 * i] = T[i].x >= kFloor;
          lv[2 * i + 1] = T[i].y >= kFloor;
        }
#pragma unroll
        for (int r = 0; r < kR; ++r) L0[r] = last[r];
        if (kTrack && !kLite) {
#pragma unroll kFwdUnroll
          for (int q = 0; q < cnt; ++q) blend_splat_spec_track<kP>(rec[q], kk[q], u.fx, fy, lv, T, acc, last);
        } else {
          if constexpr (kSplitPath) {
#ifdef XG_BWD_STATS
            {
              bool mine = false;
#pragma unroll
              for (int i = 0; i < kP; ++i) mine |= (T[i].x >= kFloor) || (T[i].y >= kFloor);
              const unsigned al = __ballot_sync(0xffffffffu, mine);
              if (lane == 0) {
                atomicAdd(&g_fwd_stats[rec_safe ? 0 : 1], 1ull);
                atomicAdd(&g_fwd_stats[rec_safe ? 2 : 3], (unsigned long long)cnt);
                const bool top = (al & 0xffffu) != 0, bot = (al >> 16) != 0;
                atomicAdd(&g_fwd_stats[(top && bot) ? 4 : 5], 1ull);
                atomicAdd(&g_fwd_stats[6], (unsigned long long)__popc(al));
              }
            }
#endif
            if (rec_safe) {
#pragma unroll kRecUnroll
              for (int q = 0; q < cnt; ++q) blend_splat_spec_rec<kP>(rh[q], u.fx, fy, T, acc);
            } else {
              blend_batch_spec<kP, kSplitUnroll>(rh, cnt, u.fx, fy, T, acc);
            }
          } else {
            blend_batch_spec<kP>(rh, cnt, u.fx, fy, T, acc);
          }
        }
        bool crossed = false;
#pragma unroll
        for (int i = 0; i < kP; ++i)
          crossed |= (T[i].x < kFloor && lv[2 * i]) || (T[i].y < kFloor && lv[2 * i + 1]);
        redo = __any_sync(0xffffffffu, crossed);
        if (redo) {
#pragma unroll
          for (int i = 0; i < kP; ++i) {
            if (kSplitPath) {
              const float4 x = sv[32 * i];
              T[i] = make_float2(x.x, x.y);
              acc[i] = make_float2(x.z, x.w);
            } else {
              T[i] = T0[i];
              acc[i] = A0[i];
            }
          }
#pragma unroll
          for (int r = 0; r < kR; ++r) last[r] = L0[r];
        }
      }
      if (redo) {
        constexpr bool kLa = kSplitPath && !kTrack;  // (image-only split records: sigma from log2 alpha)
        if (general)
          blend_batch<true, kTrack, kP, kLa>(rh, kh, cnt, u.fx, fy, T, acc, last);
        else
          blend_batch<false, kTrack, kP, kLa>(rh, kh, cnt, u.fx, fy, T, acc, last);
#pragma unroll
        for (int i = 0; i < kP; ++i) {
          if (kTrack) {
            Tf[i].x = (T[i].x < kFloor && T[i].x > 0.f) ? T[i].x : Tf[i].x;
            Tf[i].y = (T[i].y < kFloor && T[i].y > 0.f) ? T[i].y : Tf[i].y;
          }
          T[i].x = T[i].x < kFloor ? 0.f : T[i].x;
          T[i].y = T[i].y < kFloor ? 0.f : T[i].y;
        }
      }
    }
    __syncwarp();
    bool live = false;
#pragma unroll
    for (int i = 0; i < kP; ++i) live |= (T[i].x >= kFloor) || (T[i].y >= kFloor);
    alive = __any_sync(0xffffffffu, live);
  }
  if (kTma) {  // (an early-terminated warp still has copies in flight: land them before the buffers are reused)
    while (tma_ready < tma_issued - 1) tma_wait(tb, ++tma_ready);
    __syncwarp();
  }
  if (kTrack && kLite) {  // live to the end: replay from the list's last entry
    const int lend = (int)(u.end - u.start) - 1;
#pragma unroll
    for (int i = 0; i < kP; ++i) {
      if (T[i].x >= kFloor) last[2 * i] = lend;
      if (T[i].y >= kFloor) last[2 * i + 1] = lend;
    }
  }
  float l1 = 0.f;
  int wl = -1;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    if (u.px < a.w && u.py0 + r < a.h) {
      const long long o = (long long)(u.py0 + r) * a.w + u.px;
      const float v = (r & 1) ? acc[r >> 1].y : acc[r >> 1].x;
      a.image[o] = v;
      if (kTrack && a.t_final) {
        const float t = (r & 1) ? T[r >> 1].y : T[r >> 1].x, tf = (r & 1) ? Tf[r >> 1].y : Tf[r >> 1].x;
        a.t_final[o] = t > 0.f ? t : tf;
        a.n_contrib[o] = last[r] + 1;
      }
      if (a.target) l1 += fabsf(v - a.target[o]);
    }
    wl = max(wl, last[r] + 1);
  }
  if (a.target && a.l1_sum) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    if (lane == 0) atomicAdd(a.l1_sum, (double)l1);
  }
  if (kTrack && a.unit_cost) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wl = max(wl, __shfl_xor_sync(0xffffffffu, wl, o));
    // (per quarter tile: a wider sub-block records its cost for each quarter it covers)
    if (lane == 0) {
      if (kP == 1) {
        a.unit_cost[4 * tile + sub] = wl;
      } else {
        for (int q = 0; q < 4; ++q)
          if (kP == 4 || (q >> 1) == sub) a.unit_cost[4 * tile + q] = wl;
      }
    }
  }
}

// Non-persistent single-view variant: one CTA per kWarps / kSubs tiles
// (heaviest first), one warp per sub-block.
template <bool kTrack, bool kLite = false>
__global__ void __launch_bounds__(kThreads, min_ctas(fwd_pairs<kTrack, kLite>())) k_composite_fwd_np(FwdArgs a) {
  constexpr int kP = fwd_pairs<kTrack, kLite>(), kSubs = 4 / kP;
  __shared__ FRec s_rec[kWarps][kRecPerWarp];
  __shared__ int s_k[kWarps][64];
  const int warp = threadIdx.x >> 5;
  // (streamed replay: the backward grid may launch once every CTA got here;
  // it synchronises on the ring, never on this grid's completion)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const bool skip = a.n_entries && (long long)*a.n_entries > a.cap;
  const int i = blockIdx.x * (kWarps / kSubs) + warp / kSubs;
  if (!skip && i < a.n_tiles) composite_unit<kTrack, kP, kLite>(a, a.order[i], warp % kSubs, s_rec[warp], s_k[warp]);
  if (kTrack && kLite) {
    if (a.ring) {
      // publish each of the CTA's tiles' chunks (k_replay_items' count:
      // ceil(L / kCk), L = the longest replay of its quarters) after its
      // pixels, checkpoints and costs are visible; an overflowed view
      // publishes nothing
      constexpr int kTpc = kWarps / kSubs;  // tiles per CTA
      __threadfence();
      __syncthreads();
      if (threadIdx.x < kTpc) {
        uint32_t nch = 0;
        const int it = blockIdx.x * kTpc + threadIdx.x;
        const int tile = it < a.n_tiles ? a.order[it] : 0;
        if (!skip && it < a.n_tiles) {
          int L = 0;
          for (int q = 0; q < 4; ++q) L = max(L, a.unit_cost[4 * tile + q]);
          nch = (uint32_t)((L + kCk - 1) >> kCkShift);
        }
        if (nch) {
          const uint32_t p = atomicAdd(&a.ring_ctr[0], nch);
          for (uint32_t j = 0; j < nch; ++j)
            if ((long long)(p + j) < a.ring_cap) {
              const unsigned long long v = (unsigned long long)tile | ((unsigned long long)j << 20) |
                                           ((unsigned long long)a.epoch << 40);
              asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.ring + p + j), "l"(v) : "memory");
            }
        }
        __threadfence();
        if (it < a.n_tiles) atomicAdd(&a.ring_ctr[1], 1u);  // (tiles published: exactly n_tiles in the end)
      }
    }
  }
}

template <bool kTrack, bool kLite = false>
__global__ void __launch_bounds__(kThreads, min_ctas(fwd_pairs<kTrack, kLite>())) k_composite_fwd(FwdArgs a) {
  constexpr int kP = fwd_pairs<kTrack, kLite>();
  __shared__ FRec s_rec[kWarps][kRecPerWarp];
  __shared__ int s_k[kWarps][64];
  const int warp = threadIdx.x >> 5;
  int tile, sub;
  bool first = true;
  // an entry-buffer overflow leaves tile ranges past the buffer: touch nothing
  // (the caller sees XG_ST_ENTRY_OVERFLOW and re-bins the view)
  if (a.n_entries && (long long)*a.n_entries > a.cap) return;
  while (next_unit<false, 4 / kP>(a.order, a.work, a.n_tiles, first, tile, sub))
    composite_unit<kTrack, kP, kLite>(a, tile, sub, s_rec[warp], s_k[warp]);
}

// ---------------------------------------------------------------------------
// Multi-view forward (image only): one persistent launch composites up to
// kMaxBatch views of the same detector from ONE heaviest-first queue over all
// their (view, tile, quarter) units, so no view's tail leaves SMs idle and a
// launch measures the kernel alone.  Per-view buffers travel in the kernel
// parameters (no device-side table).
// ---------------------------------------------------------------------------
constexpr int kMaxBatch = 16;

struct BatchView {
  const double2* mean2d;
  const float4* coef;
  const float* inten;
  const uint32_t* entry;
  const long long* ranges;
  const uint32_t* n_entries;
  long long cap;
  float* image;
};

struct BatchArgs {
  BatchView v[kMaxBatch];
  const int* order;  // (view << 20) | tile, heaviest first over all views
  uint32_t* work;
  int n_views, n_tiles, ntx, w, h;
};

__device__ __forceinline__ bool next_batch_unit(const BatchArgs& b, bool& first, int& view, int& tile, int& quad) {
  constexpr uint32_t kSubs = 4 / kFwdPairs;
  const uint32_t n_units = kSubs * (uint32_t)(b.n_tiles * b.n_views);
  const uint32_t G = gridDim.x, w = threadIdx.x >> 5;
  const uint32_t dealt = min(n_units, G * (uint32_t)kWarps);
  uint32_t k = n_units;
  if (first) {
    first = false;
    k = G * w + ((w & 1u) ? G - 1u - blockIdx.x : blockIdx.x);
  }
  if (k >= dealt) {
    uint32_t d = 0;
    if ((threadIdx.x & 31) == 0) d = atomicAdd(b.work, 1u);
    k = dealt + __shfl_sync(0xffffffffu, d, 0);
  }
  if (k >= n_units) return false;
  const int vt = b.order[k / kSubs];
  view = vt >> 20;
  tile = vt & ((1 << 20) - 1);
  quad = (int)(k % kSubs);
  return true;
}

__global__ void __launch_bounds__(kThreads, min_ctas(kFwdPairs)) k_composite_fwd_batch(BatchArgs b) {
  __shared__ FRec s_rec[kWarps][kRecPerWarp];
  __shared__ int s_k[kWarps][32];
  const int warp = threadIdx.x >> 5;
  int view, tile, quad;
  bool first = true;
  while (next_batch_unit(b, first, view, tile, quad)) {
    const BatchView& v = b.v[view];
    if (v.n_entries && (long long)*v.n_entries > v.cap) continue;  // overflowed view: re-rendered by the caller
    FwdArgs a{v.mean2d, v.coef, v.inten, v.entry, v.ranges, nullptr, nullptr, b.n_tiles, v.image, nullptr,
              nullptr, nullptr, nullptr, nullptr, nullptr, 0, b.ntx, b.w, b.h};
    composite_unit<false, kFwdPairs>(a, tile, quad, s_rec[warp], s_k[warp]);
  }
}

// Non-persistent variant: one CTA per (view, tile), its 4 warps the tile's
// quarters, CTAs dispatched heaviest first by the hardware scheduler - as
// tiles retire, kernels from other streams (the next batch's binning, on
// higher-priority streams) fill the freed SM slots instead of waiting for the
// whole launch.
__global__ void __launch_bounds__(kThreads, min_ctas(kFwdPairs)) k_composite_fwd_batch_np(BatchArgs b) {
  constexpr int kSubs = 4 / kFwdPairs;
  __shared__ FRec s_rec[kWarps][kRecPerWarp];
  __shared__ int s_k[kWarps][32];
#if XG_FWD_TMA
  __shared__ TmaBuf s_tma[kWarps];
#endif
  const int warp = threadIdx.x >> 5;
  const int i = blockIdx.x * (kWarps / kSubs) + warp / kSubs;
  if (i >= b.n_tiles * b.n_views) return;
  const int vt = b.order[i];
  const int view = vt >> 20, tile = vt & ((1 << 20) - 1);
  const BatchView& v = b.v[view];
  if (v.n_entries && (long long)*v.n_entries > v.cap) return;
  FwdArgs a{v.mean2d, v.coef, v.inten, v.entry, v.ranges, nullptr, nullptr, b.n_tiles, v.image, nullptr,
            nullptr, nullptr, nullptr, nullptr, nullptr, 0, b.ntx, b.w, b.h};
#if XG_FWD_TMA
  composite_unit<false, kFwdPairs>(a, tile, warp % kSubs, s_rec[warp], s_k[warp], &s_tma[warp]);
#else
  composite_unit<false, kFwdPairs>(a, tile, warp % kSubs, s_rec[warp], s_k[warp]);
#endif
}

// (view, tile) pairs of a batch by descending entry count (64 log buckets).
__global__ void __launch_bounds__(1024) k_batch_tile_order(BatchArgs b, int* __restrict__ order) {
  constexpr int NB = 64;
  __shared__ int hist[NB];
  __shared__ int off[NB];
  if (threadIdx.x < NB) hist[threadIdx.x] = 0;
  __syncthreads();
  const int n = b.n_tiles * b.n_views;
  auto key = [&](int i) {
    const int vw = i / b.n_tiles, t = i - vw * b.n_tiles;
    const long long* r = b.v[vw].ranges;
    const long long len = r[2 * t + 1] - r[2 * t];
    const int bk = len > 0 ? (int)(4.f * __log2f((float)len + 1.f)) : 0;
    return NB - 1 - min(bk, NB - 1);
  };
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&hist[key(i)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int k = 0; k < NB; ++k) {
      off[k] = run;
      run += hist[k];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int vw = i / b.n_tiles, t = i - vw * b.n_tiles;
    order[atomicAdd(&off[key(i)], 1)] = (vw << 20) | t;
  }
}

// Units (quarter tiles) by descending reverse-replay cost, 64 log buckets.
__global__ void __launch_bounds__(1024) k_unit_order(const int* __restrict__ cost, int n_units,
                                                     int* __restrict__ order) {
  constexpr int NB = 64;
  __shared__ int hist[NB];
  __shared__ int off[NB];
  if (threadIdx.x < NB) hist[threadIdx.x] = 0;
  __syncthreads();
  auto key = [&](int u) {
    const int c = cost[u];
    const int b = c > 0 ? (int)(4.f * __log2f((float)c + 1.f)) : 0;
    return NB - 1 - min(b, NB - 1);
  };
  for (int u = threadIdx.x; u < n_units; u += blockDim.x) atomicAdd(&hist[key(u)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int b = 0; b < NB; ++b) {
      off[b] = run;
      run += hist[b];
    }
  }
  __syncthreads();
  for (int u = threadIdx.x; u < n_units; u += blockDim.x) order[atomicAdd(&off[key(u)], 1)] = u;
}

// Tiles by descending entry count (64 log-spaced buckets; order within a
// bucket is arbitrary - it only affects scheduling, never results).
__global__ void __launch_bounds__(1024) k_tile_order(const long long* __restrict__ ranges, int n_tiles,
                                                     int* __restrict__ order) {
  constexpr int NB = 64;
  __shared__ int hist[NB];
  __shared__ int off[NB];
  if (threadIdx.x < NB) hist[threadIdx.x] = 0;
  __syncthreads();
  auto key = [&](int t) {
    const long long len = ranges[2 * t + 1] - ranges[2 * t];
    const int b = len > 0 ? (int)(4.f * __log2f((float)len + 1.f)) : 0;
    return NB - 1 - min(b, NB - 1);
  };
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) atomicAdd(&hist[key(t)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int b = 0; b < NB; ++b) {
      off[b] = run;
      run += hist[b];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) order[atomicAdd(&off[key(t)], 1)] = t;
}

// ---------------------------------------------------------------------------
// Backward
// ---------------------------------------------------------------------------
struct BwdArgs {
  const double2* mean2d;
  const float4* coef;
  const float* inten;
  const uint32_t* entry;
  const long long* ranges;
  const int* order;
  uint32_t* work;
  int n_tiles;
  bool unit_order;  // order lists units (by reverse-replay cost) instead of tiles
  const float* t_final;
  const int* n_contrib;
  const float* dl;       // upstream dL/dI, or null -> fused L1
  const float* image;
  const float* target;
  float l1_scale;
  float* grad_acc;       // [N][8]
  const uint32_t* n_entries;  // counters[XG_CTR_ENTRIES] (or null)
  long long cap;
  int ntx, w, h;
  const float2* ckpt;         // chunked replay: the forward's checkpoints,
  const uint2* items;         //   the chunk list (tile, sub << 24 | chunk)
  const uint32_t* n_items;    //   and its length
  float* entry_grad;          // reproducible mode: per-(splat, tile) sums (plain stores), else null
  const uint32_t* slot_off;   //   splat g's slots start at slot_off[g] (exclusive scan of n_tiles)
  const ushort4* rect;        //   its tile rectangle: slot = slot_off[g] + row-major index of the tile
};

// Backward records (shared memory), signs folded as in the forward:
// every per-pixel step of the lane's two pixels is one packed FP32x2 op.
struct BRec {
  float4 a;  // mx (tile-relative), -my, A2, B2
  float4 b;  // C2, -alpha, intensity, 0
};

// Reverse step of one splat for the lane's two pixels: the gradient pass of
// _kernels.pyx:142-177 run back to front, with the suffix sum accumulated
// directly (no acc - prefix - contrib cancellation) and T restored by
// division by (1 - sigma).  Packed state: T, nS = -S (suffix sum), g.
// Produces, per pixel, nG = -(dL/dsigma * sigma) on unclamped pairs (the
// reference's g_power) and nw = -w = -(sigma T) (the caller accumulates
// the intensity gradient sum of g w with one FFMA2 per pair).
template <bool kGeneral>
__device__ __forceinline__ void unblend2(const BRec& r, float2 dy, float bdx, float adx2, bool act0, bool act1,
                                         float2 g, float2& T, float2& nS, float2& nG, float2& nw_out) {
  const float2 p = __ffma2_rn(__ffma2_rn(bc(r.b.x), dy, bc(bdx)), dy, bc(adx2));
  float2 ns = __fmul2_rn(bc(r.b.y), make_float2(ex2_approx(p.x), ex2_approx(p.y)));  // -sigma (raw)
  bool v0 = act0 & (p.x >= kCut2), v1 = act1 & (p.y >= kCut2);
  bool c0 = false, c1 = false;
  if (kGeneral) {
    v0 &= p.x <= 0.f;
    v1 &= p.y <= 0.f;
    c0 = ns.x <= -kClamp;
    c1 = ns.y <= -kClamp;
    ns.x = fmaxf(ns.x, -kClamp);
    ns.y = fmaxf(ns.y, -kClamp);
  }
  ns.x = v0 ? ns.x : 0.f;
  ns.y = v1 ? ns.y : 0.f;
  const float2 om = __fadd2_rn(bc(1.f), ns);  // 1 - sigma
  const float2 rc = make_float2(rcp_approx(om.x), rcp_approx(om.y));
  const float2 Tb = __fmul2_rn(T, rc);        // T before this splat
  const float2 nw = __fmul2_rn(ns, Tb);       // -(sigma T)
  nw_out = nw;
  const float2 in = __ffma2_rn(nS, rc, __fmul2_rn(bc(r.b.z), Tb));  // i T - S / (1 - sigma)
  const float2 dsig = __fmul2_rn(g, in);
  nG = __fmul2_rn(dsig, ns);
  nS = __ffma2_rn(bc(r.b.z), nw, nS);
  if (kGeneral) {
    if (!v0 || c0) nG.x = 0.f;
    if (!v1 || c1) nG.y = 0.f;
    T.x = v0 ? Tb.x : T.x;
    T.y = v1 ? Tb.y : T.y;
  } else {
    // an invalid pair has sigma = 0: 1 - sigma = 1, rcp.approx(1) = 1
    // exactly, so Tb = T, w = 0 and G = dsig * 0 = 0 without selects
    T = Tb;
  }
}

// The lane's 2 kP pixels (kP vertically adjacent pairs of one column,
// sharing dx and the dx-only terms) for one splat; the lane's 4 column
// partial sums {G, G dy, G dy^2, g w} and dx (negated: the caller negates the
// warp totals, which is exact).
template <bool kGeneral, int kP>
__device__ __forceinline__ bool unblend_splat(const BRec& r, int krel, float fx, const float2 (&fy)[kP],
                                              const int (&last)[2 * kP], const float2 (&g)[kP], float2 (&T)[kP],
                                              float2 (&nS)[kP], float* v, float& dxo) {
  const float dx = __fsub_rn(fx, r.a.x);
  const float adx2 = __fmul_rn(__fmul_rn(r.a.z, dx), dx);
  const float bdx = __fmul_rn(r.a.w, dx);
  float2 sG, sGdy, sGdy2, sgw;
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    const float2 dy = __fadd2_rn(fy[i], bc(r.a.y));
    float2 nG, nw;
    unblend2<kGeneral>(r, dy, bdx, adx2, krel <= last[2 * i], krel <= last[2 * i + 1], g[i], T[i], nS[i], nG,
                       nw);
    const float2 Gdy = __fmul2_rn(nG, dy);
    if (i == 0) {
      sG = nG;
      sGdy = Gdy;
      sGdy2 = __fmul2_rn(Gdy, dy);
      sgw = __fmul2_rn(g[i], nw);
    } else {
      sG = __fadd2_rn(sG, nG);
      sGdy = __fadd2_rn(sGdy, Gdy);
      sGdy2 = __ffma2_rn(Gdy, dy, sGdy2);
      sgw = __ffma2_rn(g[i], nw, sgw);
    }
  }
  v[0] = sG.x + sG.y;
  v[1] = sGdy.x + sGdy.y;
  v[2] = sGdy2.x + sGdy2.y;
  v[3] = sgw.x + sgw.y;
  dxo = dx;
  return (v[0] != 0.f) | (v[3] != 0.f);
}

// Speculative reverse step (batches of well-conditioned, alpha < 0.98999
// splats in which no pixel's last blended entry falls): no per-pair tests.
// Pixels active over the whole batch use their centre, inactive ones a row
// 1e30 away, whose p2 overflows to -inf: sigma = 0, 1 - sigma = 1,
// rcp.approx(1) = 1, so T, S and every partial stay exactly unchanged
// (G = dsig * 0 and G dy = 0 * 1e30 are zeros).  Opacity in the exponent as
// in the forward (record b.w = log2 alpha); pairs the reference skips at
// power < -30 add sigma < 9.4e-14 terms (T / (1 - sigma) == T exactly).
template <int kP>
__device__ __forceinline__ bool unblend_splat_spec(const BRec& r, float fx, const float2 (&fy)[kP],
                                                   const float2 (&g)[kP], float2 (&T)[kP], float2 (&nS)[kP],
                                                   float* v, float& dxo) {
  const float dx = __fsub_rn(fx, r.a.x);
  const float adx2 = __fmaf_rn(__fmul_rn(r.a.z, dx), dx, r.b.w);
  const float bdx = __fmul_rn(r.a.w, dx);
  float2 sG, sGdy, sGdy2, sgw;
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    const float2 dy = __fadd2_rn(fy[i], bc(r.a.y));
    const float2 p = __ffma2_rn(__ffma2_rn(bc(r.b.x), dy, bc(bdx)), dy, bc(adx2));
    const float2 ns = make_float2(-ex2_approx(p.x), -ex2_approx(p.y));  // -sigma
    const float2 om = __fadd2_rn(bc(1.f), ns);
    const float2 rc = make_float2(rcp_approx(om.x), rcp_approx(om.y));
    const float2 Tb = __fmul2_rn(T[i], rc);
    const float2 nw = __fmul2_rn(ns, Tb);
    const float2 in = __ffma2_rn(nS[i], rc, __fmul2_rn(bc(r.b.z), Tb));
    const float2 nG = __fmul2_rn(__fmul2_rn(g[i], in), ns);
    nS[i] = __ffma2_rn(bc(r.b.z), nw, nS[i]);
    T[i] = Tb;
    const float2 Gdy = __fmul2_rn(nG, dy);
    if (i == 0) {
      sG = nG;
      sGdy = Gdy;
      sGdy2 = __fmul2_rn(Gdy, dy);
      sgw = __fmul2_rn(g[i], nw);
    } else {
      sG = __fadd2_rn(sG, nG);
      sGdy = __fadd2_rn(sGdy, Gdy);
      sGdy2 = __ffma2_rn(Gdy, dy, sGdy2);
      sgw = __ffma2_rn(g[i], nw, sgw);
    }
  }
  v[0] = sG.x + sG.y;
  v[1] = sGdy.x + sGdy.y;
  v[2] = sGdy2.x + sGdy2.y;
  v[3] = sgw.x + sgw.y;
  dxo = dx;
  return (v[0] != 0.f) | (v[3] != 0.f);
}

// Sum two splats' records over the warp.  v[0..3] / v[4..7]: the lane's
// column partials {G, G dy, G dy^2, g w} of splat A / B, dxA / dxB its column
// offsets.  Lanes l and l ^ 16 share a column (make_unit, make_sub), so the
// first transpose step adds the column's two row groups (lanes < 16 keep A,
// the others B); each lane then expands its splat's column sums with its dx
// into the 8-value record {G dx, G dy, G dx^2, G dx dy, G dy^2, g w, G, 0}
// and the 16-lane transpose-reduce finishes it: lane l ends with the total
// of value (l >> 1) & 7 of splat l >> 4 (12 shuffles for two splats instead
// of 16 with the dx products formed before the reduction).
__device__ __forceinline__ float warp_reduce_cols(float (&v)[8], float dxA, float dxB) {
  const int lane = threadIdx.x & 31;
  const bool up16 = lane & 16;
  float c[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = up16 ? v[i] : v[i + 4];
    const float keep = up16 ? v[i + 4] : v[i];
    c[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  const float dx = up16 ? dxB : dxA;
  float w[8];
  w[0] = c[0] * dx;
  w[1] = c[1];
  w[2] = w[0] * dx;
  w[3] = c[1] * dx;
  w[4] = c[2];
  w[5] = c[3];
  w[6] = c[0];
  w[7] = 0.f;
  {
    const bool up = lane & 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float send = up ? w[i] : w[i + 4];
      const float keep = up ? w[i + 4] : w[i];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  {
    const bool up = lane & 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float send = up ? w[i] : w[i + 2];
      const float keep = up ? w[i + 2] : w[i];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
  }
  {
    const bool up = lane & 2;
    const float send = up ? w[0] : w[1];
    const float keep = up ? w[1] : w[0];
    w[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  w[0] += __shfl_xor_sync(0xffffffffu, w[0], 1);
  return w[0];
}

template <bool kRepro = false>
__device__ __forceinline__ int compact_bwd(const Raw& raw, int krel, const Unit& u, BRec* s_rec, int* s_k,
                                           uint32_t* s_gid, bool& general) {
  BRec r;
  bool keep = false, gen = false;
  if (raw.valid) {
    const float mx = (float)(raw.m.x - (double)u.x0), my = (float)(raw.m.y - (double)u.y0);
    const float A = raw.c.x, B = raw.c.y, C = raw.c.z, alpha = raw.c.w;
    keep = overlaps(mx, my, A, B, C, u.xa, u.xb, u.ya, u.yb);
    gen = !(alpha < kNoClampAlpha) || !well_conditioned(A, B, C);
    r.a = make_float4(mx, -my, A, B);
    r.b = make_float4(C, -alpha, raw.it, __log2f(alpha));
  }
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  general = __any_sync(0xffffffffu, keep && gen);
  if (keep) {
    const int pos = __popc(bal & lanemask_lt());
    s_rec[pos] = r;
    s_k[pos] = krel;
    // (reproducible replay: the splat's slot for this tile instead of its id)
    s_gid[pos] = kRepro ? raw.off + (uint32_t)((u.y0 / kTile - raw.r.y) * (raw.r.z - raw.r.x + 1) +
                                               (u.x0 / kTile - raw.r.x))
                        : raw.g;
  }
  __syncwarp();
  return __popc(bal);
}

// Per-splat accumulators (grad_acc[N][8]), per (pixel, entry) pair with
// G = dL/dsigma * sigma (unclamped pairs) and w = sigma T:
//   {sum G dx, sum G dy, sum G dx^2, sum G dx dy, sum G dy^2, sum g w, sum G, 0}
// xg_preprocess_bwd turns them into the reference's g_mean / g_conic /
// g_int / g_alpha using the splat's own (A2, B2, C2, alpha).  Each warp
// reduces its 64 pixels per splat and issues two vector reductions.
// kMode: 0 exact fast path, 1 general (clamp, p2 <= 0 test), 2 speculative
template <int kMode, int kP>
__device__ __forceinline__ bool unblend_any(const BRec& r, int krel, float fx, const float2 (&fy)[kP],
                                            const int (&last)[2 * kP], const float2 (&g)[kP], float2 (&T)[kP],
                                            float2 (&nS)[kP], float* v, float& dx) {
  if (kMode == 2) return unblend_splat_spec<kP>(r, fx, fy, g, T, nS, v, dx);
  return unblend_splat<kMode == 1, kP>(r, krel, fx, fy, last, g, T, nS, v, dx);
}

template <int kMode, int kP, bool kRepro>
__device__ __forceinline__ void unblend_batch(const BRec* rec, const int* kk, const uint32_t* gid, int cnt, float fx,
                                              const float2 (&fy)[kP], const int (&last)[2 * kP],
                                              const float2 (&g)[kP], float2 (&T)[kP], float2 (&nS)[kP],
                                              float* grad_acc, float* slots) {
  const int lane = threadIdx.x & 31;
  // splats two at a time, back to front (A = q, then B = q - 1), their
  // records reduced together
  for (int q = cnt - 1; q >= 0; q -= 2) {
    const bool hasB = q >= 1;
    float v[8], dxA, dxB = 0.f;
    bool any = unblend_any<kMode, kP>(rec[q], kk[q], fx, fy, last, g, T, nS, v, dxA);
    if (hasB) {
      any |= unblend_any<kMode, kP>(rec[q - 1], kk[q - 1], fx, fy, last, g, T, nS, v + 4, dxB);
    } else {
#pragma unroll
      for (int i = 4; i < 8; ++i) v[i] = 0.f;
    }
    if (!__any_sync(0xffffffffu, any)) continue;
    const float tot = -warp_reduce_cols(v, dxA, dxB);
    // value i sits in lanes 2i, 2i+1: lanes 0/8 collect A's 0-3 / 4-7,
    // lanes 16/24 collect B's
    const float t1 = __shfl_down_sync(0xffffffffu, tot, 2);
    const float t2 = __shfl_down_sync(0xffffffffu, tot, 4);
    const float t3 = __shfl_down_sync(0xffffffffu, tot, 6);
    if ((lane & 7) == 0 && (lane < 16 || hasB)) {
      if (kRepro) {
        // reproducible mode: this warp is the only writer of the (splat,
        // tile) sum (whole-tile sub-block, one chunk); it lands in the
        // splat's own slot for this tile (compact_bwd<true>), and
        // xg_reduce_entry_grads adds a splat's slots in order
        const uint32_t slot = lane < 16 ? gid[q] : gid[q - 1];
        *reinterpret_cast<float4*>(slots + 8 * (long long)slot + ((lane & 8) ? 4 : 0)) = make_float4(tot, t1, t2, t3);
      } else {
        const uint32_t id = lane < 16 ? gid[q] : gid[q - 1];
        red_add_v4(grad_acc + 8 * (long long)id + ((lane & 8) ? 4 : 0), tot, t1, t2, t3);
      }
    }
  }
}

// Upstream gradient of pixel o (dL/dI, or the fused L1 sign term).
__device__ __forceinline__ float upstream(const BwdArgs& a, long long o) {
  return a.dl ? a.dl[o] : a.l1_scale * (float)((a.image[o] > a.target[o]) - (a.image[o] < a.target[o]));
}

#ifdef XG_BWD_STATS
__device__ unsigned long long g_bwd_stats[6];
#endif

// speculative reverse batches (unblend_splat_spec)
#ifndef XG_BWD_SPEC
#define XG_BWD_SPEC 1
#endif
constexpr bool kBwdSpec = XG_BWD_SPEC != 0;

// Walk entries [e_lo, e_hi) of the tile starting at `start` back to front in
// batches of 32 ([b1 - 32, b1)), with the two-stage prefetch (entry indices
// one batch ahead of the records).
template <int kP, bool kRepro = false>
__device__ __forceinline__ void replay_range(const BwdArgs& a, const Unit& u, long long start, long long e_lo,
                                             long long e_hi, const float2 (&fy)[kP], const int (&last)[2 * kP],
                                             const float2 (&g)[kP], float2 (&T)[kP], float2 (&nS)[kP], BRec* rec,
                                             int* kk, uint32_t* gid) {
  const int lane = threadIdx.x & 31;
  const ushort4* const rr = kRepro ? a.rect : nullptr;
  const uint32_t* const ro = kRepro ? a.slot_off : nullptr;
  Raw nxt = fetch(e_hi - 32 + lane >= e_lo ? entry_at(a.entry, e_hi - 32 + lane, e_hi) : 0u,
                  e_hi - 32 + lane >= e_lo, a.mean2d, a.coef, a.inten, rr, ro);
  uint32_t g_nxt = e_hi - 64 + lane >= e_lo ? entry_at(a.entry, e_hi - 64 + lane, e_hi) : 0u;
  for (long long b1 = e_hi; b1 > e_lo; b1 -= 32) {
    const Raw cur = nxt;
    bool general;
    const int cnt = compact_bwd<kRepro>(cur, (int)(b1 - 32 - start) + lane, u, rec, kk, gid, general);
    const long long kn = b1 - 64 + lane;
    nxt = fetch(g_nxt, kn >= e_lo, a.mean2d, a.coef, a.inten, rr, ro);
    g_nxt = kn - 32 >= e_lo ? entry_at(a.entry, kn - 32, e_hi) : 0u;
    bool exact = general || !kBwdSpec;
    float2 fye[kP];
    if (!exact) {
      // every pixel active (last >= the batch's top entry) or inactive
      // (last < its bottom entry) over the whole batch: speculative step
      const int khi = (int)(b1 - 1 - start), klo = (int)(max(b1 - 32, e_lo) - start);
      bool straddle = false;
#pragma unroll
      for (int i = 0; i < kP; ++i) {
        const int l0 = last[2 * i], l1 = last[2 * i + 1];
        straddle |= (l0 >= klo && l0 < khi) || (l1 >= klo && l1 < khi);
        fye[i] = make_float2(l0 >= khi ? fy[i].x : 1e30f, l1 >= khi ? fy[i].y : 1e30f);
      }
      exact = __any_sync(0xffffffffu, straddle);
    }
#ifdef XG_BWD_STATS
    // (development aid: batches / survivors by path -> xg_debug_bwd_stats)
    if ((threadIdx.x & 31) == 0) {
      const int path = general ? 1 : exact ? 0 : 2;
      atomicAdd(&g_bwd_stats[path], 1ull);
      atomicAdd(&g_bwd_stats[3 + path], (unsigned long long)cnt);
    }
#endif
    if (general)
      unblend_batch<1, kP, kRepro>(rec, kk, gid, cnt, u.fx, fy, last, g, T, nS, a.grad_acc, a.entry_grad);
    else if (exact)
      unblend_batch<0, kP, kRepro>(rec, kk, gid, cnt, u.fx, fy, last, g, T, nS, a.grad_acc, a.entry_grad);
    else
      unblend_batch<2, kP, kRepro>(rec, kk, gid, cnt, u.fx, fye, last, g, T, nS, a.grad_acc, a.entry_grad);
    __syncwarp();
  }
}

// One (tile, quarter) unit of the reverse replay, whole, from the final state.
__device__ __forceinline__ void bwd_unit(const BwdArgs& a, int tile, int quad, BRec* rec, int* kk, uint32_t* gid) {
  const Unit u = make_unit(tile, quad, a.ntx, a.w, a.h, a.ranges);
  const long long o0 = (long long)u.py0 * a.w + u.px, o1 = o0 + a.w;
  float2 T[1] = {make_float2(0.f, 0.f)}, g[1] = {make_float2(0.f, 0.f)}, nS[1] = {make_float2(0.f, 0.f)};
  int last[2] = {-1, -1};
  if (u.in0) {
    T[0].x = a.t_final[o0];
    last[0] = a.n_contrib[o0] - 1;
    g[0].x = upstream(a, o0);
  }
  if (u.in1) {
    T[0].y = a.t_final[o1];
    last[1] = a.n_contrib[o1] - 1;
    g[0].y = upstream(a, o1);
  }
  if (g[0].x == 0.f) last[0] = -1;  // zero upstream contributes nothing: skip the replay
  if (g[0].y == 0.f) last[1] = -1;
  int wl = max(last[0], last[1]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wl = max(wl, __shfl_xor_sync(0xffffffffu, wl, o));
  const float2 fy[1] = {make_float2(u.fy0, u.fy1)};
  replay_range<1>(a, u, u.start, u.start, u.start + wl + 1, fy, last, g, T, nS, rec, kk, gid);
}

// One chunk of the checkpointed replay: entries [kCk j, kCk (j + 1)) of a
// 16-wide, 4 kP-row sub-block of the tile (2 kP pixels per lane: column
// lane & 15, rows 2 kP (lane >> 4) + 0 .. 2 kP - 1), restarted from the
// forward's checkpoint before entry kCk (j + 1) - or, for a pixel whose last
// blended entry precedes it, from its final state, which is the same state.
// The suffix sum restarts as acc_K - image (S = image - acc_K).
template <int kP, bool kRepro = false>
__device__ __forceinline__ void bwd_chunk(const BwdArgs& a, uint2 item, BRec* rec, int* kk, uint32_t* gid) {
  constexpr int kR = 2 * kP, kRows = 2 * kR;
  const int lane = threadIdx.x & 31;
  const int tile = (int)item.x, sub = (int)(item.y >> 24), j = (int)(item.y & 0xffffffu);
  Unit u;
  u.x0 = (tile % a.ntx) * kTile;
  u.y0 = (tile / a.ntx) * kTile;
  const int lx = lane & 15, ly = sub * kRows + (lane >> 4) * kR;
  u.px = u.x0 + lx;
  u.fx = (float)lx;
  u.xa = 0.f;
  u.xb = (float)(kTile - 1);
  u.ya = (float)(sub * kRows);
  u.yb = (float)(sub * kRows + kRows - 1);
  const long long start = a.ranges[2 * tile];
  float2 T[kP], g[kP], nS[kP], fy[kP];
  int last[kR];
#pragma unroll
  for (int i = 0; i < kP; ++i) {
    fy[i] = make_float2((float)(ly + 2 * i), (float)(ly + 2 * i + 1));
    nS[i] = make_float2(0.f, 0.f);
  }
  int wl = -1;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int py = u.y0 + ly + r;
    const long long o = (long long)py * a.w + u.px;
    float t = 0.f, gg = 0.f;
    int l = -1;
    if (u.px < a.w && py < a.h) {
      t = a.t_final[o];
      l = a.n_contrib[o] - 1;
      gg = upstream(a, o);
    }
    if (gg == 0.f) l = -1;
    if (r & 1) {
      T[r >> 1].y = t;
      g[r >> 1].y = gg;
    } else {
      T[r >> 1].x = t;
      g[r >> 1].x = gg;
    }
    last[r] = l;
    wl = max(wl, l);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wl = max(wl, __shfl_xor_sync(0xffffffffu, wl, o));
  const int lo = j << kCkShift, K = lo + kCk;
  const int hi = min(K, wl + 1);
  if (hi <= lo) return;
  const float2* ck = a.ckpt + 256 * ckpt_slot(start, tile, j + 1);
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    if (K <= last[r]) {
      const float2 c = ck[(ly + r) * kTile + lx];
      const float s = c.y - a.image[(long long)(u.y0 + ly + r) * a.w + u.px];
      if (r & 1) {
        T[r >> 1].y = c.x;
        nS[r >> 1].y = s;
      } else {
        T[r >> 1].x = c.x;
        nS[r >> 1].x = s;
      }
    }
  }
  replay_range<kP, kRepro>(a, u, start, start + lo, start + hi, fy, last, g, T, nS, rec, kk, gid);
}

// (no min-blocks bound: ptxas then settles at 92 registers = 5 CTAs per SM,
// measured fastest; forcing 6+ CTAs spills or slows the replay)
#ifdef XG_BWD_MIN_CTAS
__global__ void __launch_bounds__(kThreads, XG_BWD_MIN_CTAS) k_composite_bwd(BwdArgs a) {
#else
__global__ void __launch_bounds__(kThreads) k_composite_bwd(BwdArgs a) {
#endif
  __shared__ BRec s_rec[kWarps][32];
  __shared__ int s_k[kWarps][32];
  __shared__ uint32_t s_gid[kWarps][32];
  const int warp = threadIdx.x >> 5;
  BRec* rec = s_rec[warp];
  int* kk = s_k[warp];
  uint32_t* gid = s_gid[warp];
  int tile, quad;
  bool first = true;
  if (a.n_entries && (long long)*a.n_entries > a.cap) return;  // overflowed view: see k_composite_fwd
  while (a.unit_order ? next_unit<true>(a.order, a.work, a.n_tiles, first, tile, quad)
                      : next_unit<false>(a.order, a.work, a.n_tiles, first, tile, quad))
    bwd_unit(a, tile, quad, rec, kk, gid);
}

// Non-persistent variant: one single-warp CTA per unit, dispatched by the
// hardware in the forward's replay-cost order (heaviest first).
__global__ void __launch_bounds__(32) k_composite_bwd_np(BwdArgs a) {
  __shared__ BRec s_rec[32];
  __shared__ int s_k[32];
  __shared__ uint32_t s_gid[32];
  if (a.n_entries && (long long)*a.n_entries > a.cap) return;
  const int uidx = a.unit_order ? a.order[blockIdx.x] : 4 * a.order[blockIdx.x >> 2] + (int)(blockIdx.x & 3);
  bwd_unit(a, uidx >> 2, uidx & 3, s_rec, s_k, s_gid);
}

// Checkpointed replay: persistent warps over the chunk list (heaviest tiles
// first); the first wave is dealt by warp index, the rest pulled from the
// queue.  kBwdPairs pixel pairs per lane: a warp covers 16 x 4 kBwdPairs
// pixels, so the per-splat warp reduction is shared by 4 kBwdPairs pixels.
#ifndef XG_BWD_PAIRS
#define XG_BWD_PAIRS 4
#endif
constexpr int kBwdPairs = XG_BWD_PAIRS;
static_assert(kBwdPairs == 1 || kBwdPairs == 2 || kBwdPairs == 4, "a sub-block is 4, 8 or 16 rows");
constexpr int kBwdSubs = 4 / kBwdPairs;  // sub-blocks per tile

// (min 3 CTAs per SM: ptxas then keeps the atomic variant at 156 registers
// without spills; unbounded it settles at 128 registers with a 16 B spill,
// 1 % slower per C2 iteration; 4 CTAs spill more)
#ifndef XG_BWD_CK_MIN_CTAS
#define XG_BWD_CK_MIN_CTAS 3
#endif
template <bool kRepro>
__global__ void __launch_bounds__(kThreads, XG_BWD_CK_MIN_CTAS) k_composite_bwd_ck(BwdArgs a) {
  __shared__ BRec s_rec[kWarps][32];
  __shared__ int s_k[kWarps][32];
  __shared__ uint32_t s_gid[kWarps][32];
  const int warp = threadIdx.x >> 5;
  if (a.n_entries && (long long)*a.n_entries > a.cap) return;
  const uint32_t n = *a.n_items, dealt = gridDim.x * kWarps;
  uint32_t k = blockIdx.x * kWarps + warp;
  while (k < n) {
    bwd_chunk<kBwdPairs, kRepro>(a, a.items[k], s_rec[warp], s_k[warp], s_gid[warp]);
    uint32_t d = 0;
    if ((threadIdx.x & 31) == 0) d = atomicAdd(a.work, 1u);
    k = dealt + __shfl_sync(0xffffffffu, d, 0);
  }
}

// Streamed replay (xg_composite_train_pair): launched behind the training
// forward with programmatic dependent launch, so its CTAs take the SM slots
// the forward's tail leaves idle.  Warps pop ring slots in publication order
// (tiles whose forward has finished) and wait on the slot's epoch tag; once
// every tile has published, slots past the reserved count end the warp.
// Needs whole-tile chunks (kBwdPairs = 4).
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct StreamArgs {
  const unsigned long long* ring;
  long long ring_cap;
  uint32_t* ring_ctr;  // [0] reserved, [1] tiles published
  uint32_t epoch;
};

template <bool kRepro>
__global__ void __launch_bounds__(kThreads, XG_BWD_CK_MIN_CTAS) k_composite_bwd_stream(BwdArgs a, StreamArgs r) {
  static_assert(kBwdSubs == 1, "streamed chunks are whole tiles");
  __shared__ BRec s_rec[kWarps][32];
  __shared__ int s_k[kWarps][32];
  __shared__ uint32_t s_gid[kWarps][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr unsigned long long kExit = ~0ull;
  for (;;) {
    unsigned long long v = 0;
    if (lane == 0) {
      const uint32_t k = atomicAdd(a.work, 1u);
      for (;;) {
        if ((long long)k < r.ring_cap) {
          v = ld_acquire_u64(r.ring + k);
          if ((uint32_t)(v >> 40) == r.epoch) break;
        }
        if (ld_acquire_u32(r.ring_ctr + 1) >= (uint32_t)a.n_tiles) {
          const uint32_t total = *(volatile uint32_t*)r.ring_ctr;
          if ((long long)k >= r.ring_cap || k >= total) {
            v = kExit;
            break;
          }
          continue;  // (published before the last tile's count: visible now)
        }
        __nanosleep(128);
      }
    }
    v = __shfl_sync(0xffffffffu, v, 0);
    if (v == kExit) break;
    bwd_chunk<kBwdPairs, kRepro>(a, make_uint2((uint32_t)(v & 0xfffffu), (uint32_t)((v >> 20) & 0xfffffu)),
                                 s_rec[warp], s_k[warp], s_gid[warp]);
  }
}

// Chunk list of the checkpointed replay, one CTA: per tile (heaviest first,
// tile_order) and sub-block, ceil(L / kCk) chunks, L = the longest replay of
// the quarter tiles it overlaps (unit_cost, from the forward).
__global__ void __launch_bounds__(1024) k_replay_items(const int* __restrict__ cost, const int* __restrict__ order,
                                                       int n_tiles, uint2* __restrict__ items, long long cap,
                                                       uint32_t* __restrict__ n_items) {
  __shared__ uint32_t warp_tot[32];
  constexpr int kRows = 16 / kBwdSubs;
  auto chunks = [&](int t, int sub) {
    int L = 0;
    for (int rh = (sub * kRows) >> 3; rh <= (sub * kRows + kRows - 1) >> 3; ++rh)
      L = max(L, max(cost[4 * t + 2 * rh], cost[4 * t + 2 * rh + 1]));
    return (uint32_t)((L + kCk - 1) >> kCkShift);
  };
  const int per = (n_tiles + 1023) >> 10;
  const int i0 = min((int)threadIdx.x * per, n_tiles), i1 = min(i0 + per, n_tiles);
  uint32_t cnt = 0;
  for (int i = i0; i < i1; ++i)
    for (int sub = 0; sub < kBwdSubs; ++sub) cnt += chunks(order[i], sub);
  // block-wide exclusive scan of cnt
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t t = warp_tot[lane], ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    warp_tot[lane] = ti - t;
  }
  __syncthreads();
  long long off = (long long)warp_tot[w] + inc - cnt;
  for (int i = i0; i < i1; ++i) {
    const int t = order[i];
    for (int sub = 0; sub < kBwdSubs; ++sub) {
      const uint32_t nc = chunks(t, sub);
      for (uint32_t j = 0; j < nc && off < cap; ++j, ++off) items[off] = make_uint2((uint32_t)t, ((uint32_t)sub << 24) | j);
    }
  }
  if (threadIdx.x == blockDim.x - 1) *n_items = (uint32_t)min(off, cap);
}

// ---------------------------------------------------------------------------
// Launch configuration: one wave of persistent CTAs.
// ---------------------------------------------------------------------------
// CTAs per SM: the occupancy limit, or XG_*_CTAS_PER_SM (tuning knob) if set lower.
template <typename K>
int persistent_grid(K kernel, int n_units, const char* env) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  const char* e = getenv(env);
  if (e && atoi(e) > 0 && atoi(e) < per_sm) per_sm = atoi(e);
  // a full wave with the same CTA count on every SM (the dealt first wave
  // balances per CTA); tiny problems launch only what they can use
  const int grid = sms * per_sm;
  const int need = (n_units + kWarps - 1) / kWarps;
  return need < sms ? need : grid;
}

// ---------------------------------------------------------------------------
// Reference kernel-backend adapters (forward_tiles / backward_tiles).
// ---------------------------------------------------------------------------
__global__ void k_rows_to_records(long long n, const double* means, const double* conics,
                                  const double* inten, const double* opac, double2* mean2d,
                                  float4* coef, float* it) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  mean2d[i] = make_double2(means[2 * i], means[2 * i + 1]);
  coef[i] = make_float4((float)(-0.5 * kLog2e * conics[3 * i]), (float)(-kLog2e * conics[3 * i + 1]),
                        (float)(-0.5 * kLog2e * conics[3 * i + 2]), (float)opac[i]);
  it[i] = (float)inten[i];
}

__global__ void k_f32_to_f64(const float* a, double* b, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (double)a[i];
}

__global__ void k_f64_to_f32(const double* a, float* b, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}

__global__ void k_acc_to_reference(long long n, const float* acc, const float4* coef, const double* opac,
                                   double* g_mean, double* g_conic, double* g_int, double* g_alpha) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* a = acc + 8 * i;
  const float4 c = coef[i];
  const double sdx = a[0], sdy = a[1];
  g_mean[2 * i] = -kLn2 * (2.0 * c.x * sdx + (double)c.y * sdy);
  g_mean[2 * i + 1] = -kLn2 * ((double)c.y * sdx + 2.0 * c.z * sdy);
  g_conic[3 * i] = -0.5 * (double)a[2];
  g_conic[3 * i + 1] = -(double)a[3];
  g_conic[3 * i + 2] = -0.5 * (double)a[4];
  g_int[i] = (double)a[5];
  g_alpha[i] = opac[i] > 0.0 ? (double)a[6] / opac[i] : 0.0;
}

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct TilesWs {
  double2* mean2d;
  float4* coef;
  float* inten;
  float* image;
  float* t_final;
  int* n_contrib;
  float* dl;
  float* acc;
  int32_t* order;
  uint32_t* counters;
};

size_t tiles_ws(int64_t n, int32_t h, int32_t w, TilesWs* out, char* base) {
  const size_t hw = (size_t)h * (size_t)w;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off += al(bytes);
    return p;
  };
  TilesWs t;
  t.mean2d = (double2*)take(16 * (size_t)n);
  t.coef = (float4*)take(16 * (size_t)n);
  t.inten = (float*)take(4 * (size_t)n);
  t.image = (float*)take(4 * hw);
  t.t_final = (float*)take(4 * hw);
  t.n_contrib = (int*)take(4 * hw);
  t.dl = (float*)take(4 * hw);
  t.acc = (float*)take(32 * (size_t)n);
  t.order = (int32_t*)take(4 * (size_t)(((w + kTile - 1) / kTile) * ((h + kTile - 1) / kTile)));
  t.counters = (uint32_t*)take(4 * XG_NCOUNTERS);
  if (out) *out = t;
  return off + 256;
}

}  // namespace

xg_status launch_tile_order(const int64_t* ranges, int n_tiles, int32_t* order, cudaStream_t s) {
  k_tile_order<<<1, 1024, 0, s>>>((const long long*)ranges, n_tiles, order);
  return check_launch("k_tile_order");
}

}  // namespace xg

using namespace xg;

extern "C" {

// Reproducible mode: grad_acc[g] = the sum of splat g's per-tile slots
// (one per tile of its rectangle, written by exactly one warp of the reverse
// replay, zero where no pixel reached it), added in row-major tile order.
// One warp per splat: lane l reads float4 half (l & 1) of slot lo + l / 2 +
// 16 i (coalesced), sums its column in slot order, and the halves are
// combined by a fixed xor tree - a fixed summation order, so the result is
// identical run to run.
__global__ void __launch_bounds__(128) k_reduce_entry_grads(const float* __restrict__ slots,
                                                            const uint32_t* __restrict__ slot_off,
                                                            const uint32_t* __restrict__ n_tiles, long long n,
                                                            const uint32_t* n_entries, long long cap,
                                                            float* __restrict__ grad_acc) {
  const long long g = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= n) return;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!(n_entries && (long long)*n_entries > cap)) {
    const long long lo = slot_off[g], hi = lo + n_tiles[g];
    for (long long k = lo + (lane >> 1); k < hi; k += 16) {
      const float4 a = *reinterpret_cast<const float4*>(slots + 8 * k + 4 * (lane & 1));
      s.x += a.x; s.y += a.y; s.z += a.z; s.w += a.w;
    }
  }
#pragma unroll
  for (int o = 2; o < 32; o <<= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    s.z += __shfl_xor_sync(0xffffffffu, s.z, o);
    s.w += __shfl_xor_sync(0xffffffffu, s.w, o);
  }
  if (lane < 2) *reinterpret_cast<float4*>(grad_acc + 8 * g + 4 * lane) = s;
}

// reproducible-mode scratch: [slots: entry_capacity x 8 floats | slot_off: n + 1 | scan workspace]
struct EntryWs {
  float* slots;
  uint32_t* off;
  void* scan;
  size_t scan_bytes;
};

static size_t entry_ws_layout(int64_t n, int64_t cap, void* ws, EntryWs* w) {
  const size_t a = al(sizeof(float) * 8 * (size_t)(cap > 0 ? cap : 1));
  const size_t b = al(sizeof(uint32_t) * (size_t)(n + 1));
  const size_t c = scan_workspace_bytes(n + 1);
  if (w) {
    w->slots = (float*)ws;
    w->off = (uint32_t*)((char*)ws + a);
    w->scan = (char*)ws + a + b;
    w->scan_bytes = c;
  }
  return a + b + c;
}

static xg_status composite_fwd_impl(const xg_camera* cam, const xg_splats* sp, float* image, float* t_final,
                                    int32_t* n_contrib, const float* target, double* l1_sum, void* stream,
                                    bool lite) {
  if (!cam || !sp || !image || !sp->entry_splat || !sp->tile_ranges || !sp->mean2d || !sp->coef ||
      !sp->inten) {
    set_error_msg("xg_composite_fwd: invalid argument");
    return XG_ERR_INVALID;
  }
  if (!sp->tile_order || !sp->counters) {
    set_error_msg("xg_composite_fwd: tile_order / counters missing (run xg_bin_sort first)");
    return XG_ERR_INVALID;
  }
  const int n_tiles = tiles_x(*cam) * tiles_y(*cam);
  uint32_t* work = sp->counters + XG_CTR_QUEUE;
  cudaMemsetAsync(work, 0, sizeof(uint32_t), (cudaStream_t)stream);
  FwdArgs a{(const double2*)sp->mean2d, (const float4*)sp->coef, sp->inten, sp->entry_splat,
            (const long long*)sp->tile_ranges, sp->tile_order, work, n_tiles, image, t_final, n_contrib,
            target, l1_sum, (t_final && n_contrib) ? sp->unit_cost : nullptr,
            sp->entry_capacity > 0 ? sp->counters + XG_CTR_ENTRIES : nullptr, (long long)sp->entry_capacity,
            tiles_x(*cam), cam->width, cam->height,
            (t_final && n_contrib) ? (float2*)sp->replay_ckpt : nullptr};
  // grid: one CTA per tile dispatched heaviest first (non-persistent) vs the
  // persistent queue - measured: non-persistent 3 % faster for the tracked
  // (training) forward at C2, persistent 5 % faster image-only at C3;
  // XG_FWD_NONPERSISTENT=0/1 forces either
  const char* npe = getenv("XG_FWD_NONPERSISTENT");
  const bool track_np = npe ? atoi(npe) > 0 : true;
  const bool image_np = npe ? atoi(npe) > 0 : false;
#ifndef XG_FWD_ALWAYS_TRACK
  if (!t_final || !n_contrib) {  // image only: no contributor tracking
    if (image_np)
      k_composite_fwd_np<false><<<div_up(n_tiles, kWarps * kFwdPairs / 4), kThreads, 0, (cudaStream_t)stream>>>(a);
    else
      k_composite_fwd<false><<<persistent_grid(k_composite_fwd<false>, 4 / kFwdPairs * n_tiles, "XG_FWD_CTAS_PER_SM"),
                               kThreads, 0, (cudaStream_t)stream>>>(a);
    return check_launch("k_composite_fwd");
  }
#endif
  const int np_grid = div_up(n_tiles, kWarps * kFwdTrackPairs / 4);
  if (lite && track_np)
    k_composite_fwd_np<true, true><<<div_up(n_tiles, kWarps * kFwdLitePairs / 4), kThreads, 0, (cudaStream_t)stream>>>(a);
  else if (lite)
    k_composite_fwd<true, true><<<persistent_grid(k_composite_fwd<true, true>, 4 / kFwdLitePairs * n_tiles,
                                                  "XG_FWD_CTAS_PER_SM"),
                                  kThreads, 0, (cudaStream_t)stream>>>(a);
  else if (track_np)
    k_composite_fwd_np<true><<<np_grid, kThreads, 0, (cudaStream_t)stream>>>(a);
  else
    k_composite_fwd<true><<<persistent_grid(k_composite_fwd<true>, 4 / kFwdTrackPairs * n_tiles, "XG_FWD_CTAS_PER_SM"),
                            kThreads, 0, (cudaStream_t)stream>>>(a);
  return check_launch("k_composite_fwd");
}

xg_status xg_composite_fwd(const xg_camera* cam, const xg_splats* sp, float* image, float* t_final,
                           int32_t* n_contrib, const float* target, double* l1_sum, void* stream) {
  return composite_fwd_impl(cam, sp, image, t_final, n_contrib, target, l1_sum, stream, false);
}

xg_status xg_composite_fwd_train(const xg_camera* cam, const xg_splats* sp, float* image, float* t_final,
                                 int32_t* n_contrib, const float* target, double* l1_sum, void* stream) {
  if (!t_final || !n_contrib) {
    set_error_msg("xg_composite_fwd_train: t_final and n_contrib are required");
    return XG_ERR_INVALID;
  }
  return composite_fwd_impl(cam, sp, image, t_final, n_contrib, target, l1_sum, stream, true);
}

// The trainer's forward + fused-L1 reverse replay as one stream segment
// (xg_composite_fwd_train then xg_composite_bwd with dl_dimage = NULL): the
// forward publishes each finished tile's replay chunks to a device ring and
// the backward, launched with programmatic dependent launch, replays them
// while the forward's heaviest tiles are still running - no k_replay_items,
// no idle SMs in the forward's tail, no launch boundary.  Same arithmetic
// per chunk as the sequential pair (gradients agree up to float-atomic
// summation order, which is already run-dependent).  XG_TRAIN_STREAM=0
// runs the sequential pair.
xg_status xg_composite_train_pair(const xg_camera* cam, const xg_splats* sp, float* image, float* t_final,
                                  int32_t* n_contrib, const float* target, double* l1_sum, float l1_scale,
                                  float* grad_acc, void* stream) {
  if (!cam || !sp || !image || !t_final || !n_contrib || !target || !grad_acc) {
    set_error_msg("xg_composite_train_pair: invalid argument");
    return XG_ERR_INVALID;
  }
  static const bool on = !(getenv("XG_TRAIN_STREAM") && atoi(getenv("XG_TRAIN_STREAM")) == 0);
  const int n_tiles = tiles_x(*cam) * tiles_y(*cam);
  const bool ok = on && kBwdPairs == 4 && sp->replay_ckpt &&
                  sp->replay_items && sp->unit_cost && sp->tile_order && sp->counters && sp->entry_splat &&
                  sp->tile_ranges && sp->mean2d && sp->coef && sp->inten &&
                  sp->replay_slots >= xg_replay_slots(sp->entry_capacity, n_tiles);
  if (!ok) {
    xg_status st = xg_composite_fwd_train(cam, sp, image, t_final, n_contrib, target, l1_sum, stream);
    if (st != XG_OK) return st;
    return xg_composite_bwd(cam, sp, t_final, n_contrib, nullptr, image, target, l1_scale, grad_acc, stream);
  }
  // slot tag: 23-bit call counter with bit 23 set (a sequential-path chunk
  // list in the same buffer never has it); the ring is cleared per call as
  // well, so neither stale slots nor the allocation's garbage can pass as
  // published chunks
  static std::atomic<uint32_t> epochs{0};
  const uint32_t epoch = ((epochs.fetch_add(1u) + 1u) & 0x7fffffu) | 0x800000u;
  cudaStream_t s = (cudaStream_t)stream;
  // everything the pair needs zeroed happens before the forward, so the two
  // kernels are adjacent in the stream: queue head, ring reserved count,
  // tiles published (counters 5-7) and the gradient accumulator
  if (sp->n > 0) cudaMemsetAsync(grad_acc, 0, sizeof(float) * 8 * (size_t)sp->n, s);
  cudaMemsetAsync(sp->counters + XG_CTR_QUEUE, 0, 3 * sizeof(uint32_t), s);
  unsigned long long* ring = (unsigned long long*)sp->replay_items;
  const long long ring_cap = 4 * (long long)sp->replay_slots;
  cudaMemsetAsync(ring, 0, sizeof(unsigned long long) * (size_t)ring_cap, s);
  FwdArgs a{(const double2*)sp->mean2d, (const float4*)sp->coef, sp->inten, sp->entry_splat,
            (const long long*)sp->tile_ranges, sp->tile_order, sp->counters + XG_CTR_QUEUE, n_tiles, image, t_final,
            n_contrib, target, l1_sum, sp->unit_cost,
            sp->entry_capacity > 0 ? sp->counters + XG_CTR_ENTRIES : nullptr, (long long)sp->entry_capacity,
            tiles_x(*cam), cam->width, cam->height, (float2*)sp->replay_ckpt, ring, ring_cap,
            sp->counters + XG_CTR_ITEMS, epoch};
  k_composite_fwd_np<true, true><<<div_up(n_tiles, kWarps * kFwdLitePairs / 4), kThreads, 0, s>>>(a);
  xg_status st = check_launch("k_composite_fwd_np");
  if (st != XG_OK) return st;
  BwdArgs b{(const double2*)sp->mean2d, (const float4*)sp->coef, sp->inten, sp->entry_splat,
            (const long long*)sp->tile_ranges, nullptr, sp->counters + XG_CTR_QUEUE, n_tiles, false, t_final,
            n_contrib, nullptr, image, target, l1_scale, grad_acc,
            sp->entry_capacity > 0 ? sp->counters + XG_CTR_ENTRIES : nullptr, (long long)sp->entry_capacity,
            tiles_x(*cam), cam->width, cam->height, (const float2*)sp->replay_ckpt, nullptr, nullptr, nullptr,
            nullptr, nullptr};
  StreamArgs r{ring, ring_cap, sp->counters + XG_CTR_ITEMS, epoch};
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(persistent_grid(k_composite_bwd_stream<false>, 4 * n_tiles, "XG_BWD_CTAS_PER_SM"));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_composite_bwd_stream<false>, b, r);
  return check_launch("k_composite_bwd_stream");
}

size_t xg_composite_batch_workspace_bytes(const xg_camera* cam, int32_t n_views) {
  if (!cam || n_views < 1) return 256;
  return al(sizeof(int32_t) * (size_t)n_views * (size_t)(tiles_x(*cam) * tiles_y(*cam))) + 256 + 256;
}

xg_status xg_composite_fwd_batch(const xg_camera* cams, const xg_splats* sps, float* const* images,
                                 int32_t n_views, void* workspace, size_t workspace_bytes, void* stream) {
  if (!cams || !sps || !images || !workspace || n_views < 1 || n_views > kMaxBatch) {
    set_error_msg("xg_composite_fwd_batch: invalid argument (1 <= n_views <= XG_MAX_BATCH)");
    return XG_ERR_INVALID;
  }
  if (workspace_bytes < xg_composite_batch_workspace_bytes(cams, n_views)) {
    set_error_msg("xg_composite_fwd_batch: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  BatchArgs b{};
  const xg_camera& c0 = cams[0];
  for (int i = 0; i < n_views; ++i) {
    const xg_splats* sp = sps + i;
    if (cams[i].width != c0.width || cams[i].height != c0.height || !images[i] || !sp->entry_splat ||
        !sp->tile_ranges || !sp->mean2d || !sp->coef || !sp->inten) {
      set_error_msg("xg_composite_fwd_batch: views must share the detector size and be binned");
      return XG_ERR_INVALID;
    }
    b.v[i] = BatchView{(const double2*)sp->mean2d, (const float4*)sp->coef, sp->inten, sp->entry_splat,
                       (const long long*)sp->tile_ranges,
                       sp->entry_capacity > 0 && sp->counters ? sp->counters + XG_CTR_ENTRIES : nullptr,
                       (long long)sp->entry_capacity, images[i]};
  }
  b.n_views = n_views;
  b.n_tiles = tiles_x(c0) * tiles_y(c0);
  b.ntx = tiles_x(c0);
  b.w = c0.width;
  b.h = c0.height;
  int* order = (int*)workspace;
  uint32_t* work = (uint32_t*)((char*)workspace + al(sizeof(int32_t) * (size_t)n_views * (size_t)b.n_tiles));
  b.order = order;
  b.work = work;
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(work, 0, sizeof(uint32_t), s);
  k_batch_tile_order<<<1, 1024, 0, s>>>(b, order);
  xg_status st = check_launch("k_batch_tile_order");
  if (st != XG_OK) return st;
  // measured: the non-persistent grid (one CTA per (view, tile), dispatched
  // heaviest first by the hardware) beats the persistent queue by ~2 %;
  // XG_BATCH_NONPERSISTENT=0 selects the persistent kernel
  static const bool np = !(getenv("XG_BATCH_NONPERSISTENT") && atoi(getenv("XG_BATCH_NONPERSISTENT")) == 0);
  if (np) {
    k_composite_fwd_batch_np<<<div_up(b.n_tiles * n_views, kWarps * kFwdPairs / 4), kThreads, 0, s>>>(b);
    return check_launch("k_composite_fwd_batch_np");
  }
  k_composite_fwd_batch<<<persistent_grid(k_composite_fwd_batch, 4 / kFwdPairs * b.n_tiles * n_views, "XG_FWD_CTAS_PER_SM"),
                          kThreads, 0, s>>>(b);
  return check_launch("k_composite_fwd_batch");
}

static xg_status composite_bwd_impl(const xg_camera* cam, const xg_splats* sp, const float* t_final,
                                    const int32_t* n_contrib, const float* dl_dimage, const float* image,
                                    const float* target, float l1_scale, float* grad_acc, float* entry_grad,
                                    const uint32_t* slot_off, void* stream) {
  if (!cam || !sp || !t_final || !n_contrib || !(grad_acc || entry_grad) || (!dl_dimage && (!image || !target))) {
    set_error_msg("xg_composite_bwd: invalid argument");
    return XG_ERR_INVALID;
  }
  if (!sp->tile_order || !sp->counters) {
    set_error_msg("xg_composite_bwd: tile_order / counters missing (run xg_bin_sort first)");
    return XG_ERR_INVALID;
  }
  const int n_tiles = tiles_x(*cam) * tiles_y(*cam);
  uint32_t* work = sp->counters + XG_CTR_QUEUE;
  cudaMemsetAsync(work, 0, sizeof(uint32_t), (cudaStream_t)stream);
  // chunked replay from the forward's checkpoints (XG_BWD_CKPT=0: whole
  // quarter tiles, the path of frames without checkpoints)
  static const bool ck_env = !(getenv("XG_BWD_CKPT") && atoi(getenv("XG_BWD_CKPT")) == 0);
  if (ck_env && sp->replay_ckpt && sp->replay_items && sp->unit_cost && image) {
    if (sp->replay_slots < xg_replay_slots(sp->entry_capacity, n_tiles)) {
      set_error_msg("xg_composite_bwd: replay_slots < xg_replay_slots(entry_capacity, n_tiles)");
      return XG_ERR_INVALID;
    }
    uint32_t* n_items = sp->counters + XG_CTR_ITEMS;
    uint2* items = (uint2*)sp->replay_items;
    k_replay_items<<<1, 1024, 0, (cudaStream_t)stream>>>(sp->unit_cost, sp->tile_order, n_tiles, items,
                                                           4 * (long long)sp->replay_slots, n_items);
    xg_status st = check_launch("k_replay_items");
    if (st != XG_OK) return st;
    BwdArgs a{(const double2*)sp->mean2d, (const float4*)sp->coef, sp->inten, sp->entry_splat,
              (const long long*)sp->tile_ranges, nullptr, work, n_tiles, false, t_final, n_contrib, dl_dimage,
              image, target, l1_scale, grad_acc,
              sp->entry_capacity > 0 ? sp->counters + XG_CTR_ENTRIES : nullptr, (long long)sp->entry_capacity,
              tiles_x(*cam), cam->width, cam->height, (const float2*)sp->replay_ckpt, items, n_items,
              entry_grad, slot_off, (const ushort4*)sp->rect};
    if (entry_grad)  // reproducible: slot stores (its own instantiation, so the default path is unchanged)
      k_composite_bwd_ck<true><<<persistent_grid(k_composite_bwd_ck<true>, 4 * n_tiles, "XG_BWD_CTAS_PER_SM"),
                                 kThreads, 0, (cudaStream_t)stream>>>(a);
    else
      k_composite_bwd_ck<false><<<persistent_grid(k_composite_bwd_ck<false>, 4 * n_tiles, "XG_BWD_CTAS_PER_SM"),
                                  kThreads, 0, (cudaStream_t)stream>>>(a);
    return check_launch("k_composite_bwd_ck");
  }
  if (entry_grad) {
    set_error_msg("xg_composite_bwd_entries: needs the checkpointed replay (a tracking forward with "
                  "replay_ckpt, replay_items, unit_cost, and the image)");
    return XG_ERR_INVALID;
  }
  // schedule the reverse replay by the per-unit cost the forward recorded
  const bool by_unit = sp->unit_cost && sp->unit_order;
  if (by_unit) {
    k_unit_order<<<1, 1024, 0, (cudaStream_t)stream>>>(sp->unit_cost, 4 * n_tiles, sp->unit_order);
    xg_status st = check_launch("k_unit_order");
    if (st != XG_OK) return st;
  }
  BwdArgs a{(const double2*)sp->mean2d, (const float4*)sp->coef, sp->inten, sp->entry_splat,
            (const long long*)sp->tile_ranges, by_unit ? sp->unit_order : sp->tile_order, work, n_tiles, by_unit,
            t_final, n_contrib, dl_dimage, image, target, l1_scale, grad_acc,
            sp->entry_capacity > 0 ? sp->counters + XG_CTR_ENTRIES : nullptr, (long long)sp->entry_capacity,
            tiles_x(*cam), cam->width, cam->height};
  const char* npe = getenv("XG_BWD_NONPERSISTENT");
  if (npe && atoi(npe) > 0) {
    k_composite_bwd_np<<<4 * n_tiles, 32, 0, (cudaStream_t)stream>>>(a);
    return check_launch("k_composite_bwd_np");
  }
  k_composite_bwd<<<persistent_grid(k_composite_bwd, 4 * n_tiles, "XG_BWD_CTAS_PER_SM"), kThreads, 0, (cudaStream_t)stream>>>(a);
  return check_launch("k_composite_bwd");
}

xg_status xg_composite_bwd(const xg_camera* cam, const xg_splats* sp, const float* t_final,
                           const int32_t* n_contrib, const float* dl_dimage, const float* image,
                           const float* target, float l1_scale, float* grad_acc, void* stream) {
  if (grad_acc && sp && sp->n > 0)
    cudaMemsetAsync(grad_acc, 0, sizeof(float) * 8 * (size_t)sp->n, (cudaStream_t)stream);
  return composite_bwd_impl(cam, sp, t_final, n_contrib, dl_dimage, image, target, l1_scale, grad_acc, nullptr,
                            nullptr, stream);
}

size_t xg_entry_grad_bytes(int64_t n_splats, int64_t entry_capacity) {
  return entry_ws_layout(n_splats, entry_capacity, nullptr, nullptr);
}

xg_status xg_composite_bwd_entries(const xg_camera* cam, const xg_splats* sp, const float* t_final,
                                   const int32_t* n_contrib, const float* dl_dimage, const float* image,
                                   const float* target, float l1_scale, void* entry_ws, size_t entry_ws_bytes,
                                   void* stream) {
  if (kBwdSubs != 1) {
    set_error_msg("xg_composite_bwd_entries: built with XG_BWD_PAIRS != 4 (several writers per entry)");
    return XG_ERR_INVALID;
  }
  if (!entry_ws || !sp || sp->entry_capacity < 1 || !sp->rect || !sp->n_tiles ||
      entry_ws_bytes < xg_entry_grad_bytes(sp->n, sp->entry_capacity)) {
    set_error_msg("xg_composite_bwd_entries: invalid argument (entry_ws >= xg_entry_grad_bytes)");
    return XG_ERR_INVALID;
  }
  EntryWs w;
  entry_ws_layout(sp->n, sp->entry_capacity, entry_ws, &w);
  cudaStream_t s = (cudaStream_t)stream;
  // slots no reverse step reaches (culled, past every pixel's last) stay 0
  cudaMemsetAsync(w.slots, 0, sizeof(float) * 8 * (size_t)sp->entry_capacity, s);
  xg_status st = scan_u32(sp->n_tiles, nullptr, w.off, sp->n, nullptr, sp->n, w.off + sp->n, w.scan, w.scan_bytes, s);
  if (st != XG_OK) return st;
  return composite_bwd_impl(cam, sp, t_final, n_contrib, dl_dimage, image, target, l1_scale, nullptr, w.slots,
                            w.off, stream);
}

xg_status xg_reduce_entry_grads(const xg_camera* cam, const xg_splats* sp, const void* entry_ws,
                                size_t entry_ws_bytes, float* grad_acc, void* stream) {
  if (!cam || !sp || !entry_ws || !grad_acc || !sp->n_tiles || sp->n < 1 ||
      entry_ws_bytes < xg_entry_grad_bytes(sp->n, sp->entry_capacity)) {
    set_error_msg("xg_reduce_entry_grads: invalid argument");
    return XG_ERR_INVALID;
  }
  EntryWs w;
  entry_ws_layout(sp->n, sp->entry_capacity, const_cast<void*>(entry_ws), &w);
  k_reduce_entry_grads<<<div_up(32 * sp->n, 128), 128, 0, (cudaStream_t)stream>>>(
      w.slots, w.off, sp->n_tiles, sp->n,
      sp->entry_capacity > 0 && sp->counters ? sp->counters + XG_CTR_ENTRIES : nullptr, (long long)sp->entry_capacity,
      grad_acc);
  return check_launch("k_reduce_entry_grads");
}

int64_t xg_replay_slots(int64_t entry_capacity, int32_t n_tiles_total) {
  return (entry_capacity > 0 ? entry_capacity : 0) / kCk + (n_tiles_total > 0 ? n_tiles_total : 0) + 1;
}

size_t xg_tiles_workspace_bytes(int64_t n_splats, int32_t h, int32_t w) {
  return tiles_ws(n_splats > 0 ? n_splats : 1, h, w, nullptr, nullptr);
}

static xg_status tiles_common(int32_t h, int32_t w, const double* means2d, const double* conics,
                              const double* intensities, const double* opacities,
                              const int32_t* entry_splat, const int64_t* tile_ranges,
                              int64_t n_splats, void* workspace, size_t workspace_bytes,
                              cudaStream_t s, TilesWs& t, xg_camera& cam, xg_splats& sp) {
  if (h < 1 || w < 1 || n_splats < 0 || !tile_ranges || !workspace ||
      (n_splats > 0 && (!means2d || !conics || !intensities || !opacities || !entry_splat))) {
    set_error_msg("xg_*_tiles: invalid argument");
    return XG_ERR_INVALID;
  }
  if (workspace_bytes < xg_tiles_workspace_bytes(n_splats, h, w)) {
    set_error_msg("xg_*_tiles: workspace too small");
    return XG_ERR_WORKSPACE;
  }
  tiles_ws(n_splats > 0 ? n_splats : 1, h, w, &t, (char*)workspace);
  cam = xg_camera{};
  cam.width = w;
  cam.height = h;
  if (n_splats > 0) {
    k_rows_to_records<<<div_up(n_splats, 256), 256, 0, s>>>(n_splats, means2d, conics, intensities,
                                                            opacities, t.mean2d, t.coef, t.inten);
    xg_status st = check_launch("k_rows_to_records");
    if (st != XG_OK) return st;
  }
  sp = xg_splats{};
  sp.mean2d = (double*)t.mean2d;
  sp.coef = (float*)t.coef;
  sp.inten = t.inten;
  sp.entry_splat = (uint32_t*)entry_splat;
  sp.tile_ranges = (int64_t*)tile_ranges;
  sp.n = n_splats;
  sp.tile_order = t.order;
  sp.counters = t.counters;
  return launch_tile_order(tile_ranges, tiles_x(cam) * tiles_y(cam), t.order, s);
}

xg_status xg_forward_tiles(int32_t h, int32_t w, const double* means2d, const double* conics,
                           const double* intensities, const double* opacities,
                           const int32_t* entry_splat, int64_t n_entries,
                           const int64_t* tile_ranges, int64_t n_splats, double* image,
                           void* workspace, size_t workspace_bytes, void* stream) {
  (void)n_entries;
  cudaStream_t s = (cudaStream_t)stream;
  TilesWs t;
  xg_camera cam;
  xg_splats sp;
  xg_status st = tiles_common(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges,
                              n_splats, workspace, workspace_bytes, s, t, cam, sp);
  if (st != XG_OK) return st;
  if ((st = xg_composite_fwd(&cam, &sp, t.image, nullptr, nullptr, nullptr, nullptr, stream)) != XG_OK)
    return st;
  k_f32_to_f64<<<div_up((int64_t)h * w, 256), 256, 0, s>>>(t.image, image, (long long)h * w);
  return check_launch("k_f32_to_f64");
}

xg_status xg_backward_tiles(int32_t h, int32_t w, const double* means2d, const double* conics,
                            const double* intensities, const double* opacities,
                            const int32_t* entry_splat, int64_t n_entries,
                            const int64_t* tile_ranges, int64_t n_splats, const double* dl_dimage,
                            double* g_mean, double* g_conic, double* g_int, double* g_alpha,
                            void* workspace, size_t workspace_bytes, void* stream) {
  (void)n_entries;
  cudaStream_t s = (cudaStream_t)stream;
  TilesWs t;
  xg_camera cam;
  xg_splats sp;
  xg_status st = tiles_common(h, w, means2d, conics, intensities, opacities, entry_splat, tile_ranges,
                              n_splats, workspace, workspace_bytes, s, t, cam, sp);
  if (st != XG_OK) return st;
  if (n_splats == 0) return XG_OK;
  if (!dl_dimage || !g_mean || !g_conic || !g_int || !g_alpha) {
    set_error_msg("xg_backward_tiles: invalid argument");
    return XG_ERR_INVALID;
  }
  if ((st = xg_composite_fwd(&cam, &sp, t.image, t.t_final, t.n_contrib, nullptr, nullptr, stream)) != XG_OK)
    return st;
  const long long hw = (long long)h * w;
  k_f64_to_f32<<<div_up(hw, 256), 256, 0, s>>>(dl_dimage, t.dl, hw);
  cudaMemsetAsync(t.acc, 0, 32 * (size_t)n_splats, s);
  if ((st = xg_composite_bwd(&cam, &sp, t.t_final, t.n_contrib, t.dl, nullptr, nullptr, 0.f, t.acc,
                             stream)) != XG_OK)
    return st;
  k_acc_to_reference<<<div_up(n_splats, 256), 256, 0, s>>>(n_splats, t.acc, t.coef, opacities, g_mean,
                                                           g_conic, g_int, g_alpha);
  return check_launch("k_acc_to_reference");
}

#ifdef XG_BWD_STATS
// development aid (XG_BWD_STATS builds only): reverse-replay batches and
// survivors by path {exact, general, speculative}; reads and clears
int xg_debug_fwd_stats(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, xg::g_fwd_stats, sizeof(unsigned long long) * 8);
  static const unsigned long long zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(xg::g_fwd_stats, zero, sizeof(zero));
  return 0;
}

int xg_debug_bwd_stats(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, xg::g_bwd_stats, sizeof(unsigned long long) * 6);
  static const unsigned long long zero[6] = {0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(xg::g_bwd_stats, zero, sizeof(zero));
  return 0;
}
#endif

}  // extern "C"
