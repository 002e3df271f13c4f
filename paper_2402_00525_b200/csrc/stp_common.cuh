// Shared device definitions for the B200 hierarchical splat renderer.
//
// Geometry that decides culling and blend order (projection, Alg. 1 peak
// search, t_opt keys at every hierarchy level, the per-pixel alpha test) is
// evaluated in float64, following the reference's formulas
// (gaussian_math.py / tile_culling.py / hierarchy.py); B200 runs FP64 at half
// the FP32 rate, and only float64 decisions reproduce the float64 reference's
// tile lists and per-tile / per-pixel orders.  Sort keys are the fp32
// rounding of the fp64 depth (monotone), with equal-key runs re-ordered by the
// fp64 depth in K5, so the final order equals np.lexsort((rank, key, tile)).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/stp.h"

namespace stp {

constexpr int kTile = 16;
#ifndef STP_SORT_ITEMS
#define STP_SORT_ITEMS 16  // with the late look-back: C3 K4 0.342 vs 0.347 ms at 12 (profiles/r2ap)
#endif
constexpr int kSortPartition = 256 * STP_SORT_ITEMS;  // K4 entries per partition (256 threads)
constexpr int kScanBlockItems = 256 * 16;             // K2 counts per scan block (partials)
constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kSmRing = 64;  // K6 per-SM tile ring slots (C_SMT)

// Projected splat, one per kept Gaussian, indexed by Gaussian id; 160 B.
// The first 128-B line holds everything the pixel stage reads for one
// emitted entry (alpha, t_opt, colour), so each evaluation touches one line;
// the second holds the culling-only fields.
struct __align__(32) SplatRec {
  double mx, my;        // mean2d (pixels)                                   0
  double ca, cb;        // conic a, b                                        16
  double cc, q2;        // conic c; q'_z                                     32
  double m[6];          // camera-space M' = R inv_cov3 R^T as               48
                        // (m00, m11, m22, 2 m01, 2 m02, 2 m12)
  double q0, q1;        // q' = M' p_view (= R inv_cov3 (mean - origin)), x y 96
  float op;             // opacity                                           112
  float c0, c1, c2;     // SH colour (lower-clamped at 0)
  double inv_a, inv_c;  // 1/a, 1/c for the Alg. 1 edge searches            128
  double thr;           // log(opacity / eps): alpha >= eps <=> power <= thr  144
  int16_t rx0, rx1, ry0, ry1;  // coarse tile rect, inclusive (rasterizer.py:307-321)  152
};
static_assert(sizeof(SplatRec) == 160, "SplatRec must be 160 B");

// 256-bit read-only load (sm_100: LDG.E.256), 32-B aligned
__device__ __forceinline__ void ld256(const void* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
      : "l"(p));
}

// 256-bit store (sm_100: STG.E.256), 32-B aligned
__device__ __forceinline__ void st256(void* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d)
               : "memory");
}

__device__ __forceinline__ void st128d(void* p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void st128f(void* p, float a, float b, float c, float d) {
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

struct DevCam {
  double R[9];
  double pos[3];
  double fx, fy, cx, cy;
  double inv_fx, inv_fy;
  int W, H;
};

struct DevCfg {
  double eps, term, cap;
  double bg[3];
  double near_plane, guard, dilation, clamp;
  int q_tail, q_mid, q_head;
  int mid_center, with_depth, exact, rec_cap;
};

// Workspace counters (uint64), zeroed per frame except the epoch.
enum Counter {
  C_EPOCH = 0,
  C_BEHIND = 1,
  C_GUARD = 2,
  C_DEGEN = 3,
  C_KEPT = 4,
  C_ENTRIES = 5,
  C_TILES = 6,
  C_NONFINITE = 7,
  C_TIES = 8,
  C_ROWS = 9,       // K1: Gaussians appended to the row-culling list
  C_PART = 16,      // 8 per-pass partition counters
  C_WORK = 24,      // render work counter
  C_PROF = 32,      // 8 phase-profile accumulators (STP_PHASE_PROF builds)
  C_TILE = 40,      // render: global tile counter
  C_SCHED = 41,     // render: per-SM tile ring overrun / spin bound hit (must stay 0)
  C_STAT = 48,      // 32 work counters (STP_WORK_STATS builds)
  C_SM = 80,        // render: per-SM sub-tile counters [256]
  C_SMT = 336,      // render: per-SM tile ring [256][kSmRing] (tag<<32 | tile+2)
  C_PSTAT = C_SMT + 256 * 64,  // K1: per-SM projection stats [256][4] (behind, guard, degenerate, kept)
#ifdef STP_TAIL_PROF
  C_TAILP = C_PSTAT + 256 * 4,  // render: per-warp (start, end) globaltimer [4096][2]
  C_COUNT = C_TAILP + 4096 * 2
#else
  C_COUNT = C_PSTAT + 256 * 4
#endif
};

// ---------------------------------------------------------------------------
// Math shared by all kernels (float64).

// Branch-free float64 division / rsqrt for the normal, finite operands of the
// geometry: MUFU approximation + two Newton steps + one residual correction
// (within an ulp of the correctly rounded result).
__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

__device__ __forceinline__ double fdiv(double n, double d) {
  double r = rcp_approx(d);
  r = fma(r, fma(-d, r, 1.0), r);     // e -> e^2
  const double q = n * r;
  return fma(r, fma(-d, q, n), q);    // residual correction -> e^4
}

__device__ __forceinline__ double frsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
}

// max_points, tile_culling.py:55-88, for one splat and one closed square
// rect [xmin, xmin + w] x [ymin, ymin + w] (w = 16, 4 or 2; iw = 1/w exact).
// The two edge searches divide by (dyy * c) and (dxx * a); with dxx, dyy =
// +-w this is a multiply by 1/c (1/a) and by +-1/w, the latter exact, so the
// results match the reference's divisions up to the 1/c (1/a) rounding.
__device__ __forceinline__ void max_point(double mx, double my, double a, double b, double c,
                                          double inv_a, double inv_c, double xmin, double ymin,
                                          double w, double iw, double& ox, double& oy) {
  const double xmax = xmin + w, ymax = ymin + w;
  const bool inside_x = (mx >= xmin) & (mx <= xmax);
  const bool inside_y = (my >= ymin) & (my <= ymax);
  if (inside_x && inside_y) {
    ox = mx;
    oy = my;
    return;
  }
  const bool lo_x = mx <= 0.5 * (xmin + xmax), lo_y = my <= 0.5 * (ymin + ymax);
  const double px = lo_x ? xmin : xmax;
  const double py = lo_y ? ymin : ymax;
  const double dxx = lo_x ? w : -w, idxx = lo_x ? iw : -iw;
  const double dyy = lo_y ? w : -w, idyy = lo_y ? iw : -iw;
  const double rx = mx - px;
  const double ry = my - py;
  double t_y = (b * rx + c * ry) * inv_c * idyy;
  double t_x = (a * rx + b * ry) * inv_a * idxx;
  t_y = fmin(fmax(t_y, 0.0), 1.0);
  t_x = fmin(fmax(t_x, 0.0), 1.0);
  if (inside_x) t_y = 0.0;
  if (inside_y) t_x = 0.0;
  ox = px + t_x * dxx;
  oy = py + t_y * dyy;
}

// ---------------------------------------------------------------------------
// float64 exp(-p), p >= 0: exp(-p) = 2^-(k/64) * exp(-r), |r| <= ln2/128,
// degree-6 Taylor (error < 3e-20) and a 64-entry table of 2^(-j/64).
static __device__ const double kExp2Tab[64] = {
    0x1.0000000000000p+0, 0x1.fa7c1819e90d8p-1, 0x1.f50765b6e4540p-1, 0x1.efa1bee615a27p-1,
    0x1.ea4afa2a490dap-1, 0x1.e502ee78b3ff6p-1, 0x1.dfc97337b9b5fp-1, 0x1.da9e603db3285p-1,
    0x1.d5818dcfba487p-1, 0x1.d072d4a07897cp-1, 0x1.cb720dcef9069p-1, 0x1.c67f12e57d14bp-1,
    0x1.c199bdd85529cp-1, 0x1.bcc1e904bc1d2p-1, 0x1.b7f76f2fb5e47p-1, 0x1.b33a2b84f15fbp-1,
    0x1.ae89f995ad3adp-1, 0x1.a9e6b5579fdbfp-1, 0x1.a5503b23e255dp-1, 0x1.a0c667b5de565p-1,
    0x1.9c49182a3f090p-1, 0x1.97d829fde4e50p-1, 0x1.93737b0cdc5e5p-1, 0x1.8f1ae99157736p-1,
    0x1.8ace5422aa0dbp-1, 0x1.868d99b4492edp-1, 0x1.82589994cce13p-1, 0x1.7e2f336cf4e62p-1,
    0x1.7a11473eb0187p-1, 0x1.75feb564267c9p-1, 0x1.71f75e8ec5f74p-1, 0x1.6dfb23c651a2fp-1,
    0x1.6a09e667f3bcdp-1, 0x1.6623882552225p-1, 0x1.6247eb03a5585p-1, 0x1.5e76f15ad2148p-1,
    0x1.5ab07dd485429p-1, 0x1.56f4736b527dap-1, 0x1.5342b569d4f82p-1, 0x1.4f9b2769d2ca7p-1,
    0x1.4bfdad5362a27p-1, 0x1.486a2b5c13cd0p-1, 0x1.44e086061892dp-1, 0x1.4160a21f72e2ap-1,
    0x1.3dea64c123422p-1, 0x1.3a7db34e59ff7p-1, 0x1.371a7373aa9cbp-1, 0x1.33c08b26416ffp-1,
    0x1.306fe0a31b715p-1, 0x1.2d285a6e4030bp-1, 0x1.29e9df51fdee1p-1, 0x1.26b4565e27cddp-1,
    0x1.2387a6e756238p-1, 0x1.2063b88628cd6p-1, 0x1.1d4873168b9aap-1, 0x1.1a35beb6fcb75p-1,
    0x1.172b83c7d517bp-1, 0x1.1429aaea92de0p-1, 0x1.11301d0125b51p-1, 0x1.0e3ec32d3d1a2p-1,
    0x1.0b5586cf9890fp-1, 0x1.0874518759bc8p-1, 0x1.059b0d3158574p-1, 0x1.02c9a3e778061p-1};

// Reduction and polynomial constants in the constant bank: DFMA takes them
// as c[][] operands instead of two UMOVs per 64-bit immediate.
__constant__ double c_exp_k[9] = {
    0x1.71547652b82fep+6,  // 64 / ln2
    0x1.62e42fefa39efp-7,  // ln2 / 64 (hi)
    0x1.abc9e3b39803fp-62, // ln2 / 64 (lo)
    1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 700.0};

__device__ __forceinline__ double exp_neg(double p, const double* tab) {
  if (p > c_exp_k[8]) return 0.0;
  const double kd = rint(p * c_exp_k[0]);  // p * 64 / ln2
  const int k = (int)kd;
  double r = fma(-kd, c_exp_k[1], p);      // p - k ln2/64 (hi)
  r = fma(-kd, c_exp_k[2], r);             // (lo)
  // exp(-r), |r| <= ln2/128
  double e = c_exp_k[3];
  e = fma(e, -r, c_exp_k[4]);
  e = fma(e, -r, c_exp_k[5]);
  e = fma(e, -r, c_exp_k[6]);
  e = fma(e, -r, c_exp_k[7]);
  e = fma(e, -r, 1.0);
  e = fma(e, -r, 1.0);
  const int j = k & 63, ex = k >> 6;
  // 2^-ex by exponent construction (ex <= 1010 here)
  const double scale = __hiloint2double((1023 - ex) << 20, 0);
  return tab[j] * e * scale;
}


// a <= b ? a : b (= fmin for a non-NaN b; a NaN gives b) as one compare and
// one select: the compiler would canonicalise the ternary to fmin and expand
// it to a 5-instruction min/NaN sequence.
__device__ __forceinline__ double min_le(double a, double b) {
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\tselp.f64 %0, %1, %2, p;\n\t}"
      : "=d"(r) : "d"(a), "d"(b));
  return r;
}

// exp_neg without the p > 700 branch (the caller clamps p).  k = round(p *
// 64/ln2) via the 1.5*2^52 shifter (no FRND/F2I), and 2^-(k>>6) folded into
// the table entry's exponent field (exact: no underflow for p <= 700).
__device__ __forceinline__ double exp_neg_nb(double p, const double* tab) {
  const double sh = fma(p, c_exp_k[0], 0x1.8p52);
  const int k = __double2loint(sh);
  const double kd = sh - 0x1.8p52;
  double r = fma(-kd, c_exp_k[1], p);
  r = fma(-kd, c_exp_k[2], r);
  double e = c_exp_k[3];
  e = fma(e, -r, c_exp_k[4]);
  e = fma(e, -r, c_exp_k[5]);
  e = fma(e, -r, c_exp_k[6]);
  e = fma(e, -r, c_exp_k[7]);
  e = fma(e, -r, 1.0);
  e = fma(e, -r, 1.0);
  const double tj = tab[k & 63];
  const double ts = __hiloint2double(__double2hiint(tj) - ((k >> 6) << 20), __double2loint(tj));
  return ts * e;
}

// exp_neg_nb with shorter dependency chains (same table and polynomial):
// the lo part of the ln2/64 reduction becomes a factor exp(kd lo) = 1 + kd lo
// (|kd lo| < 1e-13) applied to the table entry in parallel, and exp(-r) - 1
// is evaluated in powers of r^2 (Estrin-like), folded into the final
// tsc * (1 + q) as one fma: 8 dependent float64 steps instead of 11.
// Host check against expl: max 2.4 ulp (exp_neg_nb: 1.9 ulp).
__device__ __forceinline__ double exp_neg_fast(double p, const double* tab) {
  const double sh = fma(p, c_exp_k[0], 0x1.8p52);
  const int k = __double2loint(sh);
  const double kd = sh - 0x1.8p52;
  const double r = fma(-kd, c_exp_k[1], p);
  const double corr = fma(kd, c_exp_k[2], 1.0);
  const double tj = tab[k & 63];
  const double ts = __hiloint2double(__double2hiint(tj) - ((k >> 6) << 20), __double2loint(tj));
  const double tsc = ts * corr;
  const double s2 = r * r;
  const double a1 = fma(-r, c_exp_k[6], c_exp_k[7]);  // 1/2 - r/6
  const double a2 = fma(-r, c_exp_k[4], c_exp_k[5]);  // 1/24 - r/120
  const double a2b = fma(s2, c_exp_k[3], a2);         // + r^2/720
  const double inner = fma(s2, a2b, a1);
  const double q = fma(s2, inner, -r);                 // exp(-r) - 1
  return fma(tsc, q, tsc);
}

// gauss2d's exponent from the halved conic (ha = a/2, hc = c/2; halving is
// exact): one multiply shorter than 0.5 * (...)
__device__ __forceinline__ double gpower_h(double ha, double b, double hc, double dx, double dy) {
  return fma(b * dx, dy, fma(hc * dy, dy, (ha * dx) * dx));
}

// exponent of gauss2d (tile_culling.py:96)
__device__ __forceinline__ double gpower(double a, double b, double c, double dx, double dy) {
  return 0.5 * (a * dx * dx + c * dy * dy) + b * dx * dy;
}

// opacity * exp(-power) >= eps  (rasterizer.py:337-338, hierarchy.py:197,99-101).
// Decided on the log side away from the boundary; within 1e-9 of it the
// reference's own product is evaluated.
__device__ __forceinline__ bool alpha_keep(double power, double thr, float op, double eps) {
  if (power > thr + 1e-9) return false;
  if (power < thr - 1e-9) return true;
  return (double)op * exp_neg(power, kExp2Tab) >= eps;
}

// rays_through_points (tile_culling.py:161-173): normalize(v @ R).
__device__ __forceinline__ void ray_dir(const DevCam& cam, double x, double y, double& d0,
                                        double& d1, double& d2) {
  const double v0 = (x - cam.cx) * cam.inv_fx;
  const double v1 = (y - cam.cy) * cam.inv_fy;
  d0 = v0 * cam.R[0] + v1 * cam.R[3] + cam.R[6];
  d1 = v0 * cam.R[1] + v1 * cam.R[4] + cam.R[7];
  d2 = v0 * cam.R[2] + v1 * cam.R[5] + cam.R[8];
  const double inv = frsqrt(d0 * d0 + d1 * d1 + d2 * d2);
  d0 *= inv;
  d1 *= inv;
  d2 *= inv;
}

// blend_depths (tile_culling.py:185-195) with ray_features (:176-182).
__device__ __forceinline__ double blend_depth(const double* m, double q0, double q1, double q2,
                                              double d0, double d1, double d2) {
  const double num = d0 * q0 + d1 * q1 + d2 * q2;
  const double den = (d0 * d0) * m[0] + (d1 * d1) * m[1] + (d2 * d2) * m[2] +
                     (2 * d0 * d1) * m[3] + (2 * d0 * d2) * m[4] + (2 * d1 * d2) * m[5];
  return fdiv(num, den);
}

// t_opt along the camera ray v = (u, w, 1), |v| = vn, from a SplatRec's
// camera-space M', q': |v| (v . q') / (v^T M' v), the same real number as
// blend_depth on the unit world ray R^T v / |v| (tile_culling.py:161-195)
__device__ __forceinline__ double key_rec(const double* m, double q0, double q1, double q2,
                                          double u, double w, double vn) {
  const double N = fma(u, q0, fma(w, q1, q2));
  const double D = fma(u, fma(m[0], u, fma(m[3], w, m[4])), fma(w, fma(m[1], w, m[5]), m[2]));
  return vn * fdiv(N, D);
}

// camera ray (u, w, 1) through a float64 image point and its length
__device__ __forceinline__ void cam_ray_i(double cx, double cy, double ifx, double ify, double x,
                                          double y, double& u, double& w, double& vn) {
  u = (x - cx) * ifx;
  w = (y - cy) * ify;
  const double vv = fma(u, u, fma(w, w, 1.0));
  vn = vv * frsqrt(vv);
}
__device__ __forceinline__ void cam_ray(const DevCam& cam, double x, double y, double& u,
                                        double& w, double& vn) {
  cam_ray_i(cam.cx, cam.cy, cam.inv_fx, cam.inv_fy, x, y, u, w, vn);
}

// t_opt of a SplatRec along the ray through a float64 image point
// (tile_culling.py:161-195 in the camera-space form)
__device__ __forceinline__ double key_rec_at(const DevCam& cam, const SplatRec& r, double x,
                                             double y) {
  double u, w, vn;
  cam_ray(cam, x, y, u, w, vn);
  return key_rec(r.m, r.q0, r.q1, r.q2, u, w, vn);
}

// Monotone fp32 sort key of a float64 depth: round-to-nearest, -0 -> +0,
// then the usual order-preserving bit flip.
__device__ __forceinline__ uint32_t depth_key(double d) {
  float f = __double2float_rn(d);
  if (f == 0.0f) f = 0.0f;
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ double shfl_d(double v, int src) {
  return __shfl_sync(kFull, v, src);
}

__device__ __forceinline__ double shfl_xor_d(double v, int m) {
  return __shfl_xor_sync(kFull, v, m);
}

// Tile-level exact cull for splat `r` at tile (tx, ty) (rasterizer.py:334-339).
__device__ __forceinline__ bool tile_survives(double mx, double my, double a, double b, double c,
                                              double inv_a, double inv_c, double thr, float op,
                                              double eps, int tx, int ty, double& ptx,
                                              double& pty) {
  max_point(mx, my, a, b, c, inv_a, inv_c, (double)(tx * kTile), (double)(ty * kTile), 16.0,
            0.0625, ptx, pty);
  return alpha_keep(gpower(a, b, c, ptx - mx, pty - my), thr, op, eps);
}

// Rects over 64 tiles whose ellipse covers well under half of them (long thin
// or faint splats) are culled row by row (row_span, k_rows_*); the others
// (large round splats fill their rect) stay on K1/K3's per-tile path, where
// their pairs share the warp's load-balanced rounds.  A heuristic (fp32, only
// K1 evaluates it and lists the Gaussian): est = ellipse area + perimeter in
// tiles.
#ifndef STP_ROWS
#define STP_ROWS 1
#endif
__device__ __forceinline__ bool use_rows(double a, double b, double c, double thr, int area) {
  if (!STP_ROWS || area <= 64) return false;
  const float fa = (float)a, fb = (float)b, fc = (float)c;
  const float D = fmaf(fa, fc, -fb * fb);
  const float T = fmaxf((float)thr, 0.f) + 1e-6f;
  if (!(D > 0.f)) return true;
  const float iD = __frcp_rn(D);
  const float hx = sqrtf(2.f * T * fc * iD), hy = sqrtf(2.f * T * fa * iD);
  const float est = 3.14159265f * 2.f * T * rsqrtf(D) * (1.f / 256.f) + (hx + hy) * 0.125f + 1.f;
  return (float)area > 2.f * est;
}

// Superset of the tile columns of tile row ty (within [rx0, rx1]) that
// tile_survives can keep, for rects too large to test tile by tile.  A kept
// tile holds its Alg. 1 point, where power <= thr + 1e-9 (alpha_keep), so it
// meets the ellipse E = {d : d^T Q d <= 2T}, Q = [[a, b], [b, c]], T = thr
// + margin.  E's x-extent over the row's band: the right boundary
// R(dy) = (-b dy + sqrt(2Ta - D dy^2)) / a (D = ac - b^2) is concave with its
// maximum at the rightmost point of E, dy = -b sqrt(2T / (cD)); L mirrors it.
// Returns lo > hi when the row cannot hold a kept tile; degenerate or
// non-finite input returns the whole row.
__device__ __forceinline__ void row_span(double mx, double my, double a, double b, double c,
                                         double thr, int ty, int rx0, int rx1, int& lo,
                                         int& hi) {
  lo = rx0;
  hi = rx1;
  const double T = thr + 1e-6 + 1e-6 * fabs(thr);
  const double D = a * c - b * b;
  if (!(D > 0.0 && a > 0.0 && c > 0.0 && T < 1e300 && mx == mx && my == my)) return;
  if (!(T > 0.0)) {
    lo = 1;
    hi = 0;
    return;
  }
  const double iD = 1.0 / D;
  const double ye = sqrt(2.0 * T * a * iD) * (1.0 + 1e-9) + 1e-9;  // |dy| on E
  double y0 = (double)(ty * kTile) - my, y1 = y0 + (double)kTile;
  y0 = fmax(y0, -ye);
  y1 = fmin(y1, ye);
  if (y0 > y1) {
    lo = 1;
    hi = 0;
    return;
  }
  const double ys = b * sqrt(2.0 * T / (c * D));  // dy of the leftmost point of E
  const double yr = fmin(fmax(-ys, y0), y1), yl = fmin(fmax(ys, y0), y1);
  const double ia = 1.0 / a;
  const double xr = (-b * yr + sqrt(fmax(2.0 * T * a - D * yr * yr, 0.0))) * ia;
  const double xl = (-b * yl - sqrt(fmax(2.0 * T * a - D * yl * yl, 0.0))) * ia;
  const double del = 1e-3 + 1e-7 * (fabs(mx) + fabs(xl) + fabs(xr));
  const double XL = mx + xl - del, XR = mx + xr + del;
  // tiles [16 tx, 16 tx + 16] meeting [XL, XR]
  const double flo = fmax(ceil(XL * (1.0 / kTile)) - 1.0, (double)rx0);
  const double fhi = fmin(floor(XR * (1.0 / kTile)), (double)rx1);
  if (!(flo <= fhi)) {
    lo = 1;
    hi = 0;
    return;
  }
  lo = (int)flo;
  hi = (int)fhi;
}

}  // namespace stp

// Host-side launchers (defined in the .cu files, called by stp_api.cu).
namespace stp {
struct Frame {
  // device pointers carved from the workspace
  SplatRec* recs;
  uint64_t* masks;        // per Gaussian: surviving tiles of a <= 64-tile coarse rect
  uint32_t* rowlist;      // ids of kept Gaussians with a > 64-tile rect (C_ROWS of them)
  double2* aux;           // per Gaussian (view z, |mean - origin|), GlobalZ only
  int globalz;            // sort mode GlobalZ (view-z keys, ordered blend)
  int sort_mode;          // STP_MODE_*
  int tile0, tile1;       // K6 tile band [tile0, tile1)
  DevCam* camp;           // device copy of `cam` (written by K0)
  uint8_t* state;
  uint32_t* counts;
  uint32_t* offsets;
  uint64_t* keys[2];      // packed entry words (ping-pong)
  uint32_t* vals;         // sorted Gaussian ids (written by K5)
  uint2* ranges;
  unsigned long long* counters;
  uint32_t* hist;         // [passes][256]
  unsigned long long* lookback;  // [passes][partitions][256]
  uint32_t* scan_scratch;
  int64_t n;
  int64_t ecap;
  int gw, gh, n_tiles;
  int passes, partitions;
  int depth_bits;         // entry word = (tile << depth_bits | truncated depth key) << id_bits | id
  int id_bits;
  int64_t* status;        // StpOutputs.status (device) or NULL: written by K5
  const double* col64;    // float64 splat colour [n,3] (XM_F64) or NULL
  DevCam cam;
  DevCfg cfg;
};

int device_sm_count();  // SMs of the current device (cached per device)
void launch_init(const Frame& f, cudaStream_t s);
void launch_preprocess(const Frame& f, const StpScene& sc, cudaStream_t s);
void launch_shade64(const Frame& f, const StpScene& sc, double* col64, cudaStream_t s);
void launch_ingest(const Frame& f, const StpSplatBatch& b, cudaStream_t s);
void launch_scan(const Frame& f, cudaStream_t s);
void launch_duplicate(const Frame& f, cudaStream_t s);
int launch_sort(const Frame& f, cudaStream_t s);  // returns the buffer holding the result
void launch_ranges(const Frame& f, int buf, cudaStream_t s);
// K6 extra modes (stp_render.cu) and the backward pass's buffers
// XM_F64: the forward render with float64 colour / depth accumulation and
// float64 outputs (StpOutputs.color64 ...), plus the sort error when asked
constexpr int XM_NONE = 0, XM_SERR = 1, XM_FWD = 2, XM_BWD = 3, XM_F64 = 4;
struct DevGrads {
  const double* upstream;  // [H,W,3] dL/d colour
  double* pix;             // [H,W,4]: float64 blended colour sum (3) + final T
  double* d_color;         // [n,3]   (indexed by Gaussian id)
  double* d_opacity;       // [n]
  double* d_mean2d;        // [n,2]
  double* d_conic;         // [n,3] (a, b, c)
};
void launch_render(const Frame& f, int buf, const StpOutputs& out, cudaStream_t s,
                   int xm = XM_NONE, const DevGrads* g = nullptr);
}  // namespace stp
