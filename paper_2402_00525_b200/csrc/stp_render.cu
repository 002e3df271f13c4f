// K6: hierarchical resort + front-to-back blend.
//
// Exact restatement of hierarchy.render_tile (hierarchy.py:27-219; contract in
// SURVEY.md Appendix A).  One warp owns a horizontally adjacent PAIR of 4x4
// sub-tiles; each sub-tile runs its own tail / mid queues (shared memory), and
// the warp's 32 lanes are its 32 pixels (lane>>4 = sub-tile, lane&15 = pixel).
// Persistent warps take (tile, pair) items; the 8 pairs of a tile go to warps
// of one SM (per-SM tile scheduling) so its splat records are fetched once.
//
//   load   : lane l evaluates bin entry pos+l against both 4x4 rects (one
//            record fetch, two float64 Alg. 1 peaks / alpha tests / t_opt),
//            hierarchy.py:190-199
//   sort   : warp bitonic network on (d4, rank) for both sub-tiles at once,
//            merged into each tail by rank counting (:200-207)
//   drain  : while len(tail) > q_tail - 32 pop 16 -> push_mid (:178-182)
//   mid    : the 16 popped entries are re-keyed at the four 2x2 rects (2 per
//            lane), lane pairs form sorted groups of 4 and each quad's groups
//            merge into its mid queue in order (rank-parallel, 8 lanes per
//            quad), popping 4 while len >= q_mid (:147-176).  Popped entries
//            go to a per-quad FIFO ring.
//   pixel  : one lane per pixel consumes its quad's ring: alpha, eps test,
//            cap, pixel-ray t_opt and the register insertion queue of q_head
//            that blends its minimum on overflow (:93-113, 81-91).  Rings
//            decouple production from consumption so both sub-tiles' pixels
//            are busy in the same rounds.
//   drain  : tail -> mids -> heads at the end of the bin (:210-217)
//
// Per sub-tile termination (:187-189) is exact: a sub-tile stops when all
// its 16 pixels have T < 1e-4 (blends of terminated pixels are no-ops, so
// stopping is output-identical).  Rects stay full size at image borders
// (hierarchy.py:124-142); pixels outside the image run as terminated.
#include <algorithm>

#include "stp_common.cuh"

namespace stp {

#ifndef STP_QT_SPECIALIZE
#define STP_QT_SPECIALIZE 1
#endif
// K6 blocks of 2 warps with a 7-block bound: ptxas still allocates 128
// registers (8 blocks = 16 warps per SM, as with 4 x 4) but schedules the
// hot loops differently; measured K6 3.580 -> 3.533 ms and the C3 view 4.29
// -> 4.23 ms (profiles/r3b, r3c: 4 x 4 at 166 regs 3.83, 2 x 7 capped at 144
// regs 3.90, 1-warp blocks 3.62-3.72, 4 x 4 by __maxnreg__(128) 3.58 ms)
#ifndef STP_EXACT_MINB
#define STP_EXACT_MINB 7
#endif
#ifndef STP_WARPS_PER_BLOCK
#define STP_WARPS_PER_BLOCK 2
#endif
constexpr int kWarpsPerBlock = STP_WARPS_PER_BLOCK;
constexpr int kRenderThreads = 32 * kWarpsPerBlock;
constexpr unsigned kNoId = 0xffffffffu;

// Warp-level strip culls in the Window / FullPerPixel and GlobalZ scans
// (strip_may_pass)
#ifndef STP_WIN_STRIP
#define STP_WIN_STRIP 1
#endif

// Optional phase profiler (-DSTP_PHASE_PROF): warp-cycles per phase are
// accumulated into counters C_PROF.. (load, merge, push_mid, pixel, items).
#ifdef STP_PHASE_PROF
#define PROF_T0() long long _pt = clock64()
#define PROF_ADD(slot)                                                              \
  do {                                                                              \
    const long long _pn = clock64();                                                \
    if (lane == 0) atomicAdd(A.counters + C_PROF + (slot), (unsigned long long)(_pn - _pt)); \
    _pt = _pn;                                                                      \
  } while (0)
#else
#define PROF_T0() (void)0
#define PROF_ADD(slot) (void)0
#endif
// Optional work counters (-DSTP_WORK_STATS), separate from the phase timer
// because their ballots and atomics perturb the timing.
#ifdef STP_WORK_STATS
#define STAT_ADD(slot, pred)                                                        \
  do {                                                                              \
    const unsigned _b = __ballot_sync(kFull, (pred));                               \
    if (lane == 0 && _b) atomicAdd(A.counters + C_STAT + (slot), (unsigned long long)__popc(_b)); \
  } while (0)
// the same inside divergent code (ballot over the active lanes)
#define STAT_ADD_DIV(slot, pred)                                                    \
  do {                                                                              \
    const unsigned _m = __activemask();                                             \
    const unsigned _b = __ballot_sync(_m, (pred));                                  \
    if (lane == __ffs(_m) - 1 && _b)                                                \
      atomicAdd(A.counters + C_STAT + (slot), (unsigned long long)__popc(_b));      \
  } while (0)
#else
#define STAT_ADD(slot, pred) (void)0
#define STAT_ADD_DIV(slot, pred) (void)0
#endif

// (d, rank) order.  Non-short-circuit: the three comparisons issue in
// parallel and combine in one predicate op (a short-circuit chain costs two
// dependent float64 compares, ~16 cycles, on every compare-exchange).
__device__ __forceinline__ bool lt(double da, uint32_t ia, double db, uint32_t ib) {
  const bool l = da < db, e = da == db, li = ia < ib;
  return l | (e & li);
}

// Sort keys of the hierarchical kernel.  STP_IKEY=1: the float64 key as an
// order-preserving int64 (sign-magnitude -> two's complement: negative
// doubles flip their magnitude bits; -0 is canonicalised to +0 first, so
// int64 equality is float64 equality).  The (key, rank) order is unchanged
// bit for bit; compares run on the integer pipe instead of DSETP chains.
#ifndef STP_EXP_FAST
#define STP_EXP_FAST 0  // exp_neg_fast in the pixel stage: measured neutral-to-slower (3.59-3.63 vs 3.58 ms, profiles/r2aa)
#endif
#ifndef STP_GPOW_H
#define STP_GPOW_H 1  // pixel-stage power from the halved conic (gpower_h): K6 3.578 vs 3.592 ms (profiles/r2aa)
#endif
#ifndef STP_IKEY
#define STP_IKEY 0  // measured slower: K6 3.71 vs 3.59 ms (profiles/r2w)
#endif
#if STP_IKEY
typedef long long Key;
__device__ __forceinline__ Key dkey(double d) {
  const long long b = __double_as_longlong(d + 0.0);
  return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double kdbl(Key k) {  // the transform is an involution
  return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffLL));
}
__device__ __forceinline__ bool lt(Key a, uint32_t ia, Key b, uint32_t ib) {
  const bool l = a < b, e = a == b, li = ia < ib;
  return l | (e & li);
}
constexpr Key kInfKey = 0x7ff0000000000000LL;  // dkey(+inf)
#else
typedef double Key;
__device__ __forceinline__ Key dkey(double d) { return d; }
__device__ __forceinline__ double kdbl(Key k) { return k; }
#define kInfKey ((double)INFINITY)
#endif
__device__ __forceinline__ Key shfl_k(Key v, int src, int w = 32) {
  return __shfl_sync(kFull, v, src, w);
}
__device__ __forceinline__ Key shfl_xor_k(Key v, int m) { return __shfl_xor_sync(kFull, v, m); }

template <int QH>
struct Head {
  Key t[QH];
  double a[QH];
  uint32_t id[QH];
  int n;
};

// Extra per-blend work of a K6 instantiation (template int XM):
//   XM_NONE  the forward render
//   XM_SERR  + the sort error delta (metrics.py:46-73)
//   XM_FWD   + the float64 blended colour sum and final T per pixel (the
//            backward pass's first replay)
//   XM_BWD   the backward replay (gradients.py:103-162): the same blend order
//            recomputed, each contribution's gradients scattered
//   XM_F64   + float64 colour / depth sums, float64 outputs composited over
//            the background in float64 (the reference's output precision),
//            and the sort error when StpOutputs.sort_error is set

struct Pixel {
  double px, py;
  double u, w, vn;    // camera ray (u, w, 1) of the pixel centre, |(u, w, 1)|
                      // (rasterizer.py:405 in the camera-space form)
  double T;           // transmittance (float64: the termination test)
  float C0, C1, C2, D;
  int rc;             // blend records written
  int64_t pix;        // y * W + x, -1 outside the image
  double tprev, serr; // XM_SERR: last blended t, sum of positive inversions
  double f0, f1, f2;  // XM_FWD: sum of colour * w; XM_BWD: that sum (full)
  double a0, a1, a2;  // XM_BWD: running sum (acc)
  double g0, g1, g2;  // XM_BWD: upstream dL/dcolour of the pixel
  double tn;          // XM_BWD: the pixel's final T
  double dd;          // XM_F64: float64 depth sum
};

struct RenderArgs {
  const SplatRec* __restrict__ recs;
  const uint32_t* __restrict__ vals;
  const uint2* __restrict__ ranges;
  DevCam cam;
  DevCfg cfg;
  int gw, n_items;
  int tile0;              // first tile of the band (items are band-relative)
  float log_eps;
  StpOutputs out;
  unsigned long long* counters;
  DevGrads grad;          // XM_FWD / XM_BWD
  const double* col64;    // XM_F64: float64 splat colour [n,3] or NULL
};

// per-pixel state of the extra modes at the start of a pixel
template <int XM>
__device__ __forceinline__ void xm_init(Pixel& P, const RenderArgs& A) {
  P.tprev = -INFINITY;
  P.serr = 0.0;
  P.f0 = P.f1 = P.f2 = 0.0;
  P.a0 = P.a1 = P.a2 = 0.0;
  P.g0 = P.g1 = P.g2 = 0.0;
  P.tn = 0.0;
  P.dd = 0.0;
  if (XM == XM_BWD && P.pix >= 0) {
    const double* g = A.grad.upstream + P.pix * 3;
    P.g0 = g[0];
    P.g1 = g[1];
    P.g2 = g[2];
    const double* q = A.grad.pix + P.pix * 4;
    P.f0 = q[0];
    P.f1 = q[1];
    P.f2 = q[2];
    P.tn = q[3];
  }
}

// gradients of one blended contribution (gradients.py:124-162, the
// front-to-back form: trailing colour = full - acc - term)
__device__ __noinline__ void bwd_step(Pixel& P, const RenderArgs& A, double al, uint32_t id,
                                      float4 oc) {
  const double T = P.T, w = al * T;
  const double c0 = oc.y, c1 = oc.z, c2 = oc.w;
  P.a0 += c0 * w;
  P.a1 += c1 * w;
  P.a2 += c2 * w;
  const double om = fmax(1.0 - al, 1e-6);
  const double d_alpha = P.g0 * (c0 * T - (P.f0 - P.a0 + A.cfg.bg[0] * P.tn) / om) +
                         P.g1 * (c1 * T - (P.f1 - P.a1 + A.cfg.bg[1] * P.tn) / om) +
                         P.g2 * (c2 * T - (P.f2 - P.a2 + A.cfg.bg[2] * P.tn) / om);
  if (!isfinite(d_alpha)) atomicAdd(A.counters + C_NONFINITE, 1ull);
  atomicAdd(A.grad.d_color + id * 3 + 0, P.g0 * w);
  atomicAdd(A.grad.d_color + id * 3 + 1, P.g1 * w);
  atomicAdd(A.grad.d_color + id * 3 + 2, P.g2 * w);
  if (al < A.cfg.cap) {
    const SplatRec& r = A.recs[id];
    const double dx = P.px - r.mx, dy = P.py - r.my;
    atomicAdd(A.grad.d_opacity + id, d_alpha * (al / (double)oc.x));
    const double da = d_alpha * al;
    atomicAdd(A.grad.d_mean2d + id * 2 + 0, da * (r.ca * dx + r.cb * dy));
    atomicAdd(A.grad.d_mean2d + id * 2 + 1, da * (r.cb * dx + r.cc * dy));
    atomicAdd(A.grad.d_conic + id * 3 + 0, -da * 0.5 * dx * dx);
    atomicAdd(A.grad.d_conic + id * 3 + 1, -da * dx * dy);
    atomicAdd(A.grad.d_conic + id * 3 + 2, -da * 0.5 * dy * dy);
  }
}

// the extra work of one blended contribution (before T is updated)
template <int XM>
__device__ __forceinline__ void xm_step(Pixel& P, const RenderArgs& A, double t, double al,
                                        uint32_t id, float4 oc) {
  if (XM == XM_SERR || XM == XM_F64) {
    P.serr += fmax(P.tprev - t, 0.0);
    P.tprev = t;
  }
  if (XM == XM_F64 && A.col64) {
    const double w = al * P.T;
    const double* c = A.col64 + (size_t)id * 3;
    P.f0 += c[0] * w;
    P.f1 += c[1] * w;
    P.f2 += c[2] * w;
  } else if (XM == XM_FWD || XM == XM_F64) {
    const double w = al * P.T;
    P.f0 += (double)oc.y * w;
    P.f1 += (double)oc.z * w;
    P.f2 += (double)oc.w * w;
  } else if (XM == XM_BWD) {
    bwd_step(P, A, al, id, oc);
  }
}

// per-pixel outputs of the extra modes at the end of a pixel
template <int XM>
__device__ __forceinline__ void xm_done(const Pixel& P, const RenderArgs& A) {
  if (P.pix < 0) return;
  if (XM == XM_SERR) A.out.sort_error[P.pix] = (float)P.serr;
  if (XM == XM_F64) {
    if (A.out.sort_error) A.out.sort_error[P.pix] = (float)P.serr;
    double* c = A.out.color64 + P.pix * 3;
    c[0] = P.f0 + P.T * A.cfg.bg[0];
    c[1] = P.f1 + P.T * A.cfg.bg[1];
    c[2] = P.f2 + P.T * A.cfg.bg[2];
    if (A.out.transmittance64) A.out.transmittance64[P.pix] = P.T;
    if (A.out.depth64) A.out.depth64[P.pix] = P.dd;
  }
  if (XM == XM_FWD) {
    double* q = A.grad.pix + P.pix * 4;
    q[0] = P.f0;
    q[1] = P.f1;
    q[2] = P.f2;
    q[3] = P.T;
  }
}

// debug blend-record capture (cold path, kept out of line)
__device__ __noinline__ void write_record(StpOutputs out, int cap, int64_t pix, int rc, double t,
                                          double al, uint32_t id) {
  if (rc < cap && pix >= 0) {
    const int64_t o = pix * cap + rc;
    out.rec_splat[o] = (int32_t)id;
    out.rec_t[o] = (float)t;
    out.rec_alpha[o] = (float)al;
    if (out.rec_t64) out.rec_t64[o] = t;
    if (out.rec_alpha64) out.rec_alpha64[o] = al;
  }
}

// blend (hierarchy.py:81-91)
template <int XM>
__device__ __forceinline__ void blend(Pixel& P, const RenderArgs& A, double t, double al,
                                      uint32_t id) {
  if (P.T < A.cfg.term) return;
  const float4 oc = __ldg(reinterpret_cast<const float4*>(&A.recs[id].op));
  const double w = al * P.T;
  const float wf = (float)w;
  P.C0 += oc.y * wf;
  P.C1 += oc.z * wf;
  P.C2 += oc.w * wf;
  P.D += (float)(t * w);
  if (XM == XM_F64) P.dd += t * w;
  if (A.cfg.rec_cap > 0) write_record(A.out, A.cfg.rec_cap, P.pix, P.rc++, t, al, id);
  xm_step<XM>(P, A, t, al, id, oc);
  P.T = P.T * (1.0 - al);
}

// blend of a live pixel (P.T >= term checked by the caller)
template <int XM>
__device__ __forceinline__ void blend_live(Pixel& P, const RenderArgs& A, double t, double al,
                                           uint32_t id) {
  const float4 oc = __ldg(reinterpret_cast<const float4*>(&A.recs[id].op));
  const double w = al * P.T;
  const float wf = (float)w;
  P.C0 += oc.y * wf;
  P.C1 += oc.z * wf;
  P.C2 += oc.w * wf;
  P.D += (float)(t * w);
  if (XM == XM_F64) P.dd += t * w;
  if (A.cfg.rec_cap > 0) write_record(A.out, A.cfg.rec_cap, P.pix, P.rc++, t, al, id);
  xm_step<XM>(P, A, t, al, id, oc);
  P.T = P.T * (1.0 - al);
}

// alpha / eps test / cap / pixel-ray t_opt of one emitted entry
// (hierarchy.py:94-105), branch-free: everything computed, the decision
// returned, so two evaluations placed side by side form one basic block
// whose float64 chains the scheduler interleaves.
__device__ __forceinline__ bool emit_eval_bf(const Pixel& P, const RenderArgs& A, uint32_t id,
                                             const double* tab, double& t, double& al) {
  const SplatRec* r = A.recs + id;
  // the record's first 128-B line in four 256-bit loads
  double mx, my, a, b, c, q2, m0, m1, m2, m3, m4, m5, q0, q1, opc, c12;
  ld256(&r->mx, mx, my, a, b);
  ld256(&r->cc, c, q2, m0, m1);
  ld256(&r->m[2], m2, m3, m4, m5);
  ld256(&r->q0, q0, q1, opc, c12);
  const float op = __int_as_float(__double2loint(opc));
  const double dx = P.px - mx, dy = P.py - my;
#if STP_GPOW_H
  const double pw = gpower_h(0.5 * a, b, 0.5 * c, dx, dy);
#else
  const double pw = gpower(a, b, c, dx, dy);
#endif
  const double mm[6] = {m0, m1, m2, m3, m4, m5};
  t = key_rec(mm, q0, q1, q2, P.u, P.w, P.vn);
  const double pc = min_le(pw, 700.0);
#if STP_EXP_FAST
  al = (double)op * exp_neg_fast(pc, tab);
#else
  al = (double)op * exp_neg_nb(pc, tab);
#endif
  const bool pass = al >= A.cfg.eps;  // hierarchy.py:99-101
  al = min_le(al, A.cfg.cap);
  return pass;
}

// emit_eval_bf behind a conservative float32 early-out (alpha < eps beyond
// doubt, the float64 test decides everything else) for the scans of the
// Window / FullPerPixel kernel, which evaluate every bin entry at every pixel
// of a 16 x 2 strip: most entries miss the whole strip, and the warp then
// skips the t_opt division and the exp.
#ifndef STP_WIN_PRETEST
#define STP_WIN_PRETEST 1
#endif
__device__ __forceinline__ bool emit_eval_pre(const Pixel& P, const RenderArgs& A, uint32_t id,
                                              const double* tab, double& t, double& al) {
#if STP_WIN_PRETEST
  const SplatRec* r = A.recs + id;
  double mx, my, a, b;
  ld256(&r->mx, mx, my, a, b);
  const double c = __ldg(&r->cc);
  const float op = __ldg(&r->op);
  const double pw = gpower_h(0.5 * a, b, 0.5 * c, P.px - mx, P.py - my);
  const float thr = __logf(op) - A.log_eps;
  if ((float)pw > thr + fmaf(1e-5f, fabsf(thr), 1e-5f)) return false;
#endif
  return emit_eval_bf(P, A, id, tab, t, al);
}

// insort into the pixel queue; on overflow blend the minimum
// (hierarchy.py:110-113).  Branch-free: empty slots hold (+inf, ~0), the
// overflow case blends min(e, H[0]) and, if H[0] left, shifts the queue and
// re-inserts e; insertion is a compare-and-select bubble over the slots.
// EXACT: the queue size equals QH; else runtime qh <= QH.
template <int QH, bool EXACT, int XM>
__device__ __forceinline__ void head_push(Pixel& P, Head<QH>& H, const RenderArgs& A, int qh_rt,
                                          Key t, double al, uint32_t id) {
  const int qh = EXACT ? QH : qh_rt;
  const bool full = H.n >= qh;
  if (EXACT && full) {
    // c[i] = e < H[i] is monotone in i (H sorted).  The blended entry is
    // min(e, H[0]); the new queue is R[i] = c[i] ? H[i] : (c[i+1] ? e :
    // H[i+1]), R[QH-1] = c[QH-1] ? H[QH-1] : e (unchanged when c[0]).  All
    // compares issue in parallel, no branch.  The caller checked P.T >= term.
    bool c[QH];
#pragma unroll
    for (int i = 0; i < QH; ++i) c[i] = lt(t, id, H.t[i], H.id[i]);
    blend_live<XM>(P, A, kdbl(c[0] ? t : H.t[0]), c[0] ? al : H.a[0], c[0] ? id : H.id[0]);
#pragma unroll
    for (int i = 0; i < QH; ++i) {
      const bool nx = i + 1 < QH;
      const int j = nx ? i + 1 : i;
      const bool cn = nx ? c[j] : false;
      H.t[i] = c[i] ? H.t[i] : (cn ? t : (nx ? H.t[j] : t));
      H.a[i] = c[i] ? H.a[i] : (cn ? al : (nx ? H.a[j] : al));
      H.id[i] = c[i] ? H.id[i] : (cn ? id : (nx ? H.id[j] : id));
    }
    return;
  }
  if (full) {
    const bool e_min = lt(t, id, H.t[0], H.id[0]);
    blend<XM>(P, A, kdbl(e_min ? t : H.t[0]), e_min ? al : H.a[0], e_min ? id : H.id[0]);
    if (e_min) return;
    // drop H[0], insert e at position c among H[1..qh-1]
    int c = 0;
#pragma unroll
    for (int i = 1; i < QH; ++i)
      if ((EXACT || i < qh) && lt(H.t[i], H.id[i], t, id)) ++c;
#pragma unroll
    for (int i = 0; i < QH; ++i) {
      const int j = (i + 1 < QH) ? i + 1 : i;
      const bool take_next = i < c;
      const bool take_e = i == c;
      H.t[i] = take_next ? H.t[j] : (take_e ? t : H.t[i]);
      H.a[i] = take_next ? H.a[j] : (take_e ? al : H.a[i]);
      H.id[i] = take_next ? H.id[j] : (take_e ? id : H.id[i]);
    }
    return;
  }
  H.n++;
  Key xt = t;
  double xa = al;
  uint32_t xi = id;
#pragma unroll
  for (int i = 0; i < QH; ++i) {
    const bool sw = lt(xt, xi, H.t[i], H.id[i]);
    const Key ht = H.t[i];
    const double ha = H.a[i];
    const uint32_t hi = H.id[i];
    H.t[i] = sw ? xt : ht;
    H.a[i] = sw ? xa : ha;
    H.id[i] = sw ? xi : hi;
    xt = sw ? ht : xt;
    xa = sw ? ha : xa;
    xi = sw ? hi : xi;
  }
}

// Bitonic sort of two (d, id) arrays, one pair per lane each, ascending.
// Rolled loops: the kernel is instruction-fetch bound, code size matters more
// than the loop overhead here.
__device__ __forceinline__ void warp_sort2(Key& d0, uint32_t& i0, Key& d1, uint32_t& i1,
                                           int lane) {
#pragma unroll 1
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      const Key od0 = shfl_xor_k(d0, j);
      const uint32_t oi0 = __shfl_xor_sync(kFull, i0, j);
      const Key od1 = shfl_xor_k(d1, j);
      const uint32_t oi1 = __shfl_xor_sync(kFull, i1, j);
      const bool want_min = (((lane & j) == 0) == ((lane & k) == 0));
      // elements are distinct (ids unique) except empty slots, whose swap is
      // a no-op: "partner < me" decides both directions with one compare
      const bool take0 = want_min == lt(od0, oi0, d0, i0);
      const bool take1 = want_min == lt(od1, oi1, d1, i1);
      d0 = take0 ? od0 : d0;
      i0 = take0 ? oi0 : i0;
      d1 = take1 ? od1 : d1;
      i1 = take1 ? oi1 : i1;
    }
  }
}

// Bitonic sort of (d, id) within each 16-lane half of the warp (L = lane &
// 15; both halves sorted ascending at once).
__device__ __forceinline__ void half_sort16(Key& d, uint32_t& id, int L) {
#pragma unroll 1
  for (int k = 2; k <= 16; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      const Key od = shfl_xor_k(d, j);
      const uint32_t oi = __shfl_xor_sync(kFull, id, j);
      const bool want_min = (((L & j) == 0) == ((L & k) == 0));
      const bool take = want_min == lt(od, oi, d, id);
      d = take ? od : d;
      id = take ? oi : id;
    }
  }
}

// position of the k-th (0-based) set bit of m (k < popc(m))
__device__ __forceinline__ int select_bit32(unsigned m, int k) {
  int pos = 0;
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    const int c = __popc(m & ((1u << s) - 1u));
    const bool up = k >= c;
    k -= up ? c : 0;
    m = up ? (m >> s) : m;
    pos += up ? s : 0;
  }
  return pos;
}

// number of (d,id) in sorted a[0..n) strictly below (x, xi)
#ifndef STP_CB8
#define STP_CB8 0  // measured slower: K6 4.08 vs 3.60 ms (profiles/r2x)
#endif
__device__ __forceinline__ int count_below(const Key* ad, const uint32_t* ai, int n, Key x,
                                           uint32_t xi) {
#if STP_CB8
  // 8-ary search: each round issues 7 independent probes (lo + i q - 1) and
  // narrows [lo, hi) to at most q - 1 elements, so n <= 63 takes two
  // rounds of shared-memory latency instead of five dependent ones
  int lo = 0, hi = n;
  while (hi > lo) {
    const int q = (hi - lo + 8) >> 3;  // 8q > hi - lo: the range after is < q
    int k = 0;
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      const int p = lo + i * q - 1;
      const int pc = p < hi ? p : lo;
      k += (p < hi) & lt(ad[pc], ai[pc], x, xi);
    }
    const int nlo = lo + k * q;
    hi = min(hi, nlo + q - 1);
    lo = nlo;
  }
  return lo;
#else
  int lo = 0, hi = n;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (lt(ad[m], ai[m], x, xi)) lo = m + 1;
    else hi = m;
  }
  return lo;
#endif
}

// ---------------------------------------------------------------------------
// Shared-memory queues of one sub-tile, addressed arithmetically (units of
// one element: doubles in the key region, uint32 in the id region):
//   [tail qt (x2 unless qt == 64) | mid 4 x MS | scratch 4 x SS | pad |
//    groups 4 x GS]  and, ids only, [rings 4 x RS].
// The per-quad strides are odd (MS = qm+1, SS = qm+5, GS = 17, RS = R+1)
// and the group base sits 4 elements past a 16-element boundary relative to
// the mids, so the 4 quads' arrays -- read by the same instruction in the
// mid merge and the pixel stage -- fall on distinct shared-memory banks.
// The sorted load batch (<= 32) lives in the group region (groups exist only
// inside push_mid, the batch only inside a merge).  With qt == 64 a merge
// reads at most 32 + 32 entries, two per lane, so it runs in place (read and
// rank everything, then write) and the tail is single-buffered.  Shared
// memory is traded against L1: the records the warps re-read live in the
// rest of the SM's 256 KB (measured: 32 KB less L1 per SM = +5.5% K6).
#ifndef STP_RING
#define STP_RING 64
#endif
#ifndef STP_RANK16
#define STP_RANK16 1  // batch order by all-pairs ranking (else a bitonic network)
#endif
#ifndef STP_RANK_UNROLL
#define STP_RANK_UNROLL 8  // with the 2 x 7 K6 blocks: 8 + READY 12 K6 3.535 -> 3.519 ms (profiles/r3f)
#endif
constexpr int kRankUnroll = STP_RANK_UNROLL;
#ifndef STP_RING_PF
#define STP_RING_PF 1  // pixel stage: ring ids one step ahead: K6 3.516 -> 3.453 ms (profiles/r3k); 2: + L1 prefetch of those records, 3.50 ms (r3n)
#endif
#ifndef STP_SID_PF
#define STP_SID_PF 0  // 1: load-phase bin entries one batch ahead (K6 3.525 vs 3.520 ms); 2: + L2 prefetch of their records (3.537): off (profiles/r3g)
#endif
#ifndef STP_READY
#define STP_READY 12  // consume once every producing sub-tile has this many emits (16 before the 2 x 7 blocks)
#endif
__host__ __device__ inline int ring_size(int qm) { return qm <= 16 ? STP_RING : 128; }
__host__ __device__ inline bool tail_inplace(int qt) { return qt == 64; }
__host__ __device__ inline int q_mid0(int qt) { return (tail_inplace(qt) ? 1 : 2) * qt; }
__host__ __device__ inline int q_scr0(int qt, int qm) { return q_mid0(qt) + 4 * (qm + 1); }
__host__ __device__ inline int q_grp0(int qt, int qm) {
  const int b = q_scr0(qt, qm) + 4 * (qm + 5);
  return b + ((q_mid0(qt) + 4 - b) & 15);
}
__host__ __device__ inline int q_ring0(int qt, int qm) { return q_grp0(qt, qm) + 4 * 17; }
__host__ __device__ inline int sub_nd(int qt, int qm) { return q_ring0(qt, qm); }
__host__ __device__ inline int sub_ni(int qt, int qm) {
  return q_ring0(qt, qm) + 4 * (ring_size(qm) + 1);
}
__host__ __device__ inline size_t warp_smem_bytes(int qt, int qm) {
  return ((size_t)2 * sub_nd(qt, qm) * 8 + (size_t)2 * sub_ni(qt, qm) * 4 + 15) & ~(size_t)15;
}

struct SubQ {
  Key* d;
  uint32_t* i;
  int qt, qm;
  __device__ __forceinline__ Key* td(int c) const { return d + c * qt; }
  __device__ __forceinline__ uint32_t* ti(int c) const { return i + c * qt; }
  __device__ __forceinline__ Key* bd() const { return d + q_grp0(qt, qm); }
  __device__ __forceinline__ uint32_t* bi() const { return i + q_grp0(qt, qm); }
  __device__ __forceinline__ int o_mid(int q) const { return q_mid0(qt) + q * (qm + 1); }
  __device__ __forceinline__ int o_scr(int q) const { return q_scr0(qt, qm) + q * (qm + 5); }
  __device__ __forceinline__ int o_grp(int q) const { return q_grp0(qt, qm) + 17 * q; }
  __device__ __forceinline__ uint32_t* ring(int q, int R) const {
    return i + q_ring0(qt, qm) + q * (R + 1);
  }
};

// QMX = 8: mid queues of at most 8 (loops statically bounded); 0: generic.
// QT > 0: the queue sizes are compile-time (tail QT, mid QMX), so every
// shared-memory offset is an immediate (the default 64/8/4 configuration;
// otherwise the compiler re-derives the offsets inside the hot loops).
template <int QH, bool EXACT, int QMX, int QT, int XM>
#ifdef STP_K6_MAXNREG
// experiments: a register cap instead of a min-blocks bound
#define STP_K6_BOUNDS __maxnreg__(STP_K6_MAXNREG)
#else
#define STP_K6_BOUNDS __launch_bounds__(kRenderThreads, STP_EXACT_MINB)
#endif
__global__ void STP_K6_BOUNDS k_render(RenderArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_tab[64];
  const int qt = QT ? QT : A.cfg.q_tail, qm = (QT && QMX) ? QMX : A.cfg.q_mid;
  const int qh_rt = A.cfg.q_head;
  const int R = ring_size(qm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64; i += kRenderThreads) s_tab[i] = kExp2Tab[i];
  __syncthreads();
  unsigned char* wbase = smem_raw + warp * warp_smem_bytes(qt, qm);
  const int nd = sub_nd(qt, qm), ni = sub_ni(qt, qm);
  auto subq = [&](int s) {
    SubQ q;
    q.d = reinterpret_cast<Key*>(wbase) + s * nd;
    q.i = reinterpret_cast<uint32_t*>(reinterpret_cast<Key*>(wbase) + 2 * nd) + s * ni;
    q.qt = qt;
    q.qm = qm;
    return q;
  };
  const double term = A.cfg.term;
  const int drain_lim = qt - 32;  // drain_tail(q_tail - batch_load)

  // pixel role: sub-tile lane>>4, pixel lane&15 (4x4 row-major), quad
  const int ps = lane >> 4, pp = lane & 15;
  const int ppx = pp & 3, ppy = pp >> 2;
  const int pq = (ppy >> 1) * 2 + (ppx >> 1);
  // push_mid role: quad, group, half of group
  const int mq = lane >> 3, mg = (lane >> 1) & 3, mh = lane & 1;

  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  smid &= 255;
  unsigned long long* sm_cnt = A.counters + C_SM + smid;
  unsigned long long* sm_ring = A.counters + C_SMT + smid * kSmRing;

#ifdef STP_TAIL_PROF
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int gwarp = blockIdx.x * kWarpsPerBlock + warp;
#endif
  for (;;) {
    // ---- work item: (tile, pair) with the 8 pairs of a tile on one SM
    int tile = -1, pair = 0;
    if (lane == 0) {
      const unsigned long long i = atomicAdd(sm_cnt, 1ull);
      const unsigned long long tl = i >> 3;
      pair = (int)(i & 7);
      unsigned long long* slot = sm_ring + (tl % kSmRing);
      if (pair == 0) {
        const int g = (int)atomicAdd(A.counters + C_TILE, 1ull);
        const int gt = g < A.n_items ? g + A.tile0 : -1;
        atomicExch(slot, (tl << 32) | (unsigned long long)(gt + 2));
        tile = gt;
      } else {
        // pair 0 of tile tl was drawn before this pair (one counter per SM)
        // and publishes it right after its draw.  The slot could only be
        // overwritten once kSmRing more tiles start on this SM, i.e. after
        // the SM's other warps finished hundreds of items while this one did
        // not get to read: bounded and reported (C_SCHED) instead of hanging.
        unsigned long long v;
        unsigned spins = 0;
        for (;;) {
          v = *reinterpret_cast<volatile unsigned long long*>(slot);
          const unsigned long long tag = v >> 32;
          if (tag == tl && (v & 0xffffffffull) != 0) break;
          if (tag > tl || ++spins > (1u << 26)) {
            atomicAdd(A.counters + C_SCHED, 1ull);
            if (A.out.status) atomicExch(reinterpret_cast<unsigned long long*>(A.out.status),
                                         (unsigned long long)STP_ERR_CUDA);
            v = 1;  // tile -1: stop
            break;
          }
          if (spins > 64) __nanosleep(32);
        }
        tile = (int)(v & 0xffffffffull) - 2;
      }
    }
    tile = __shfl_sync(kFull, tile, 0);
    pair = __shfl_sync(kFull, pair, 0);
#ifdef STP_TAIL_PROF
    if (tile < 0 && lane == 0 && gwarp < 4096) {
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      A.counters[C_TAILP + 2 * gwarp] = t_start;
      A.counters[C_TAILP + 2 * gwarp + 1] = t_end;
    }
#endif
    if (tile < 0) break;
    const int tx = tile % A.gw, ty = tile / A.gw;
    // pair p covers sub-tiles (row p>>1, columns 2*(p&1), 2*(p&1)+1)
    const int sx0 = tx * kTile + (pair & 1) * 8, sy0 = ty * kTile + (pair >> 1) * 4;

    Pixel P;
    {
      const int gx = sx0 + ps * 4 + ppx, gy = sy0 + ppy;
      const bool in_img = gx < A.cam.W && gy < A.cam.H;
      P.pix = in_img ? (int64_t)gy * A.cam.W + gx : -1;
      P.px = (double)gx + 0.5;
      P.py = (double)gy + 0.5;
      cam_ray(A.cam, P.px, P.py, P.u, P.w, P.vn);
      P.T = in_img ? 1.0 : 0.0;
      P.C0 = P.C1 = P.C2 = P.D = 0.f;
      P.rc = 0;
      xm_init<XM>(P, A);
    }
    Head<QH> H;
    H.n = 0;
#pragma unroll
    for (int i = 0; i < QH; ++i) {
      H.t[i] = kInfKey;
      H.a[i] = 0.0;
      H.id[i] = kNoId;
    }

    const uint2 rg = A.ranges[tile];
    const int start = (int)rg.x, k_total = (int)(rg.y - rg.x);
    const double r4y = (double)sy0;
#if STP_SID_PF
    // the next load batch's bin entries, one batch ahead (the record loads
    // then wait on one global load instead of two dependent ones)
    uint32_t pf_sid = lane < k_total ? __ldg(A.vals + start + lane) : 0u;
#endif
    PROF_T0();
    PROF_ADD(5);

    // per-sub-tile pipeline state (warp-uniform scalars; s selects)
    int cur0 = 0, cur1 = 0, th0 = 0, th1 = 0, nt0 = 0, nt1 = 0, nm0 = 0, nm1 = 0;
    int rh0 = 0, rh1 = 0, rt0 = 0, rt1 = 0;
    bool prod0 = k_total > 0, prod1 = k_total > 0;  // still producing emits
    int pos = 0;

    // ---- push_mid for sub-tile s: pop c = min(16, len(tail)) entries and
    // run them through the four mid queues (hierarchy.py:147-176)
    auto push_mid = [&](int s) {
      const SubQ Q = subq(s);
      const int cur = s ? cur1 : cur0, th = s ? th1 : th0, nt = s ? nt1 : nt0;
      int nm = s ? nm1 : nm0, rt = s ? rt1 : rt0;
      const int c = min(16, nt);
      const uint32_t* tip = Q.ti(cur) + th;
      const double r2x = (double)(sx0 + 4 * s) + (mq & 1) * 2, r2y = r4y + (mq >> 1) * 2;
      Key gd[4];
      uint32_t gi[4];
      gd[0] = gd[1] = kInfKey;
      gi[0] = gi[1] = kNoId;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int e = 4 * mg + 2 * mh + u;
        if (e < c) {
          const uint32_t sid = tip[e];
          const SplatRec* r = A.recs + sid;
          // the record in 256-bit loads: everything but colour
          double mx, my, a, b, c, q2, m[6], q0, q1, x0, x1, ia, ic, x2, x3;
          ld256(&r->mx, mx, my, a, b);
          ld256(&r->cc, c, q2, m[0], m[1]);
          ld256(&r->m[2], m[2], m[3], m[4], m[5]);
          ld256(&r->q0, q0, q1, x0, x1);
          double ptx, pty;
          if (A.cfg.mid_center) {
            ptx = r2x + 1.0;
            pty = r2y + 1.0;
          } else {
            ld256(&r->inv_a, ia, ic, x2, x3);
            max_point(mx, my, a, b, c, ia, ic, r2x, r2y, 2.0, 0.5, ptx, pty);
          }
          double cu, cw, cv;
          cam_ray(A.cam, ptx, pty, cu, cw, cv);
          const Key dv = dkey(key_rec(m, q0, q1, q2, cu, cw, cv));
          if (u) {
            gd[1] = dv;
            gi[1] = sid;
          } else {
            gd[0] = dv;
            gi[0] = sid;
          }
        }
      }
      gd[2] = shfl_xor_k(gd[0], 1);
      gi[2] = __shfl_xor_sync(kFull, gi[0], 1);
      gd[3] = shfl_xor_k(gd[1], 1);
      gi[3] = __shfl_xor_sync(kFull, gi[1], 1);
#define CSWAP(a, b)                                        \
  if (lt(gd[b], gi[b], gd[a], gi[a])) {                    \
    const Key td_ = gd[a]; gd[a] = gd[b]; gd[b] = td_;      \
    const uint32_t ti_ = gi[a]; gi[a] = gi[b]; gi[b] = ti_; \
  }
      CSWAP(0, 1) CSWAP(2, 3) CSWAP(0, 2) CSWAP(1, 3) CSWAP(1, 2)
#undef CSWAP
      Key* gdp = Q.d + Q.o_grp(mq);
      uint32_t* gip = Q.i + Q.o_grp(mq);
      // lane half mh stores sorted slots 2mh, 2mh+1 (selects: no local memory)
      gdp[4 * mg + 2 * mh] = mh ? gd[2] : gd[0];
      gip[4 * mg + 2 * mh] = mh ? gi[2] : gi[0];
      gdp[4 * mg + 2 * mh + 1] = mh ? gd[3] : gd[1];
      gip[4 * mg + 2 * mh + 1] = mh ? gi[3] : gi[1];
      __syncwarp();
      Key* md = Q.d + Q.o_mid(mq);
      uint32_t* mi = Q.i + Q.o_mid(mq);
      Key* sd = Q.d + Q.o_scr(mq);
      uint32_t* si = Q.i + Q.o_scr(mq);
      uint32_t* ring = Q.ring(mq, R);
      const int slot0 = lane & 7;
      for (int gg = 0; 4 * gg < c; ++gg) {
        const int ng = min(4, c - 4 * gg);
        const Key* g_d = gdp + 4 * gg;
        const uint32_t* g_i = gip + 4 * gg;
        STAT_ADD(10, (lane & 7) == 0);                                        // mid merges
        STAT_ADD(11, (lane & 7) == 0 && QMX == 8 && qm == 8 && nm == 4 && ng == 4);  // steady
        if (QMX == 8 && qm == 8 && nm == 4 && ng == 4) {
          // steady state: mid holds 4, a full group of 4 arrives, the merged 8
          // emit their first 4 and keep the last 4.  Lane slot sl owns one
          // element: its rank = index + #(other list < it), 4 comparisons.
          const bool from_mid = slot0 < 4;
          const int ix = slot0 & 3;
          const Key x = from_mid ? md[ix] : g_d[ix];
          const uint32_t xi = from_mid ? mi[ix] : g_i[ix];
          const Key* od = from_mid ? g_d : md;
          const uint32_t* oi = from_mid ? g_i : mi;
#ifdef STP_WORK_STATS
          {  // merges that are appends (the group sorts after the mid queue)
            const bool app = lt(md[3], mi[3], g_d[0], g_i[0]);
            const bool all_app = __all_sync(kFull, app);
            STAT_ADD(20, slot0 == 0 && app);
            STAT_ADD(21, lane == 0 && all_app);
          }
#endif
          int rk = ix;
#pragma unroll
          for (int u = 0; u < 4; ++u) rk += lt(od[u], oi[u], x, xi);
          __syncwarp();
          if (rk < 4) ring[(rt + rk) & (R - 1)] = xi;
          else {
            md[rk - 4] = x;
            mi[rk - 4] = xi;
          }
          rt += 4;
          __syncwarp();
          continue;
        }
        const int L = nm + ng;
#pragma unroll 1
        for (int k = 0; k < 1; ++k) {
#pragma unroll 1
          for (int sl = slot0; sl < L; sl += 8) {
            Key x;
            uint32_t xi;
            int rk;
            if (sl < nm) {
              x = md[sl];
              xi = mi[sl];
              rk = sl;
#pragma unroll 1
              for (int u = 0; u < ng; ++u) rk += lt(g_d[u], g_i[u], x, xi);
            } else {
              x = g_d[sl - nm];
              xi = g_i[sl - nm];
              rk = sl - nm;
#pragma unroll 1
              for (int u = 0; u < nm; ++u) rk += lt(md[u], mi[u], x, xi);
            }
            sd[rk] = x;
            si[rk] = xi;
          }
        }
        __syncwarp();
        const int h0 = (L >= qm) ? 4 : 0;  // flush_mid pops 4 (:168-176)
#pragma unroll 1
        for (int sl = slot0; sl < L; sl += 8) {
          if (sl < h0) ring[(rt + sl) & (R - 1)] = si[sl];
          else {
            md[sl - h0] = sd[sl];
            mi[sl - h0] = si[sl];
          }
        }
        rt += h0;
        nm = L - h0;
        __syncwarp();
      }
      if (s) {
        th1 += c;
        nt1 -= c;
        nm1 = nm;
        rt1 = rt;
      } else {
        th0 += c;
        nt0 -= c;
        nm0 = nm;
        rt0 = rt;
      }
    };

    // Scheduling (any order is output-identical: each sub-tile's queues see
    // exactly its own entry stream and each pixel its quad's emit stream):
    //  - consume when every producing sub-tile has >= 16 pending emits (both
    //    halves of the warp busy), or a ring is nearly full;
    //  - otherwise produce: tails over the drain limit pop first (before any
    //    load, as drain_tail follows every batch), then the next batch is
    //    loaded for both sub-tiles, and at the end of the bin mids flush.
    const int ring_full = R - 16 - qm;
    for (;;) {
      const int pa = rt0 - rh0, pb = rt1 - rh1;
      const bool ready = (!prod0 || pa >= STP_READY) && (!prod1 || pb >= STP_READY);
      if (pa > ring_full || pb > ring_full || (ready && pa + pb > 0)) {
        // ================= consume: pixels take emits from their quad rings
        const int rounds = (pa > 0 && pb > 0) ? min(pa, pb) : max(pa, pb);
        STAT_ADD(9, lane == 0);
        {
          const int pend = ps ? pb : pa;
          const int base = ps ? rh1 : rh0;
          const uint32_t* ring = subq(ps).ring(pq, R);
          // STP_PIX_UNROLL emitted entries per step: their evaluations are
          // independent (one basic block, interleaved chains); the head
          // insertions stay in order.  Terminated pixels skip the insertion (their blends are
          // no-ops, hierarchy.py:82-84).
#ifndef STP_PIX_UNROLL
#define STP_PIX_UNROLL 2
#endif
#if STP_RING_PF
          // the next step's ring ids one step ahead (the record loads then
          // start without waiting on the shared-memory load)
          const int lim1 = max(min(pend, rounds) - 1, 0);
          uint32_t nid[STP_PIX_UNROLL];
#pragma unroll
          for (int k = 0; k < STP_PIX_UNROLL; ++k) nid[k] = ring[(base + min(k, lim1)) & (R - 1)];
#endif
          for (int e = 0; e < rounds; e += STP_PIX_UNROLL) {
            const int lim = min(pend, rounds);
            const bool live = P.T >= term;
            uint32_t ids[STP_PIX_UNROLL];
#if STP_RING_PF
#pragma unroll
            for (int k = 0; k < STP_PIX_UNROLL; ++k) {
              ids[k] = nid[k];
              nid[k] = ring[(base + min(e + STP_PIX_UNROLL + k, lim1)) & (R - 1)];
            }
#if STP_RING_PF > 1
            if (e + STP_PIX_UNROLL < lim && live) {
#pragma unroll
              for (int k = 0; k < STP_PIX_UNROLL; ++k) {
                const char* rp = reinterpret_cast<const char*>(A.recs + nid[k]);
                asm volatile("prefetch.global.L1 [%0];" ::"l"(rp));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + 96));
              }
            }
#endif
#endif
            double ts[STP_PIX_UNROLL], as[STP_PIX_UNROLL];
            bool ps[STP_PIX_UNROLL];
#ifdef STP_WORK_STATS
            bool evk[STP_PIX_UNROLL], fk[STP_PIX_UNROLL];
#pragma unroll
            for (int k = 0; k < STP_PIX_UNROLL; ++k) evk[k] = fk[k] = false;
#endif
            if (e < lim && live) {
#pragma unroll
              for (int k = 0; k < STP_PIX_UNROLL; ++k) {
                const bool vk = e + k < lim;
#if !STP_RING_PF
                ids[k] = ring[(base + e + (vk ? k : 0)) & (R - 1)];
#endif
                ps[k] = emit_eval_bf(P, A, ids[k], s_tab, ts[k], as[k]) & vk;
#ifdef STP_WORK_STATS
                evk[k] = vk;
                fk[k] = vk && !ps[k];
#endif
              }
#pragma unroll
              for (int k = 0; k < STP_PIX_UNROLL; ++k) {
#ifdef STP_WORK_STATS
                {  // head pushes onto a full queue; those sorting after every queued entry
                  const bool doit = ps[k] && P.T >= term, fullq = H.n >= QH;
                  const bool aft = !lt(ts[k], ids[k], H.t[QH - 1], H.id[QH - 1]);
                  STAT_ADD_DIV(16, doit && fullq);
                  STAT_ADD_DIV(17, doit && fullq && aft);
                  const unsigned m_ = __activemask();
                  const unsigned bd_ = __ballot_sync(m_, doit && fullq);
                  const unsigned bn_ = __ballot_sync(m_, doit && fullq && !aft);
                  STAT_ADD_DIV(18, lane == __ffs(m_) - 1 && bd_ != 0);
                  STAT_ADD_DIV(19, lane == __ffs(m_) - 1 && bd_ != 0 && bn_ == 0);
                }
#endif
                // (a warp-uniform "sorts after the whole queue" shortcut --
                // 92% of full-queue pushes -- measured slower: 3.86 vs 3.59
                // ms, profiles/r2o; the select network is cheaper than the
                // vote + second code path)
                if (ps[k] && P.T >= term)
                  head_push<QH, EXACT, XM>(P, H, A, qh_rt, dkey(ts[k]), as[k], ids[k]);
              }
            }
#ifdef STP_WORK_STATS
            STAT_ADD(8, lane == 0);
#pragma unroll
            for (int k = 0; k < STP_PIX_UNROLL; ++k) {
              STAT_ADD(4, e + k < pend);
              STAT_ADD(5, evk[k]);
              STAT_ADD(6, evk[k] && !fk[k]);
              // quad lanes: base b, b+1, b+4, b+5; all slots of live quad
              // lanes failed (terminated lanes count as failed)
              const unsigned bf = __ballot_sync(kFull, fk[k] || (e + k < pend && !evk[k]));
              const unsigned bv = __ballot_sync(kFull, e + k < pend);
              const int qb = (lane & 16) + (pq >> 1) * 8 + (pq & 1) * 2;
              const unsigned qmask = 0x33u << qb;
              STAT_ADD(7, evk[k] && (bf & qmask) == qmask && (bv & qmask) == qmask);
            }
#endif
          }
        }
        rh0 += min(rounds, pa);
        rh1 += min(rounds, pb);
        __syncwarp();
        PROF_ADD(3);
        continue;
      }
      if (!prod0 && !prod1) break;  // nothing pending, nothing to produce
      // ================= produce
      const int lim = (pos < k_total) ? drain_lim : 0;
      const bool over0 = prod0 && nt0 > lim, over1 = prod1 && nt1 > lim;
      if (over0 || over1) {
        push_mid((over0 && (!over1 || pa <= pb)) ? 0 : 1);
        PROF_ADD(2);
        continue;
      }
      if (pos < k_total) {
        // ---- termination check per sub-tile (hierarchy.py:187-189)
        const unsigned bal = __ballot_sync(kFull, P.T < term);
        if (prod0 && (bal & 0xffffu) == 0xffffu) {
          prod0 = false;
          rh0 = rt0;
        }
        if (prod1 && (bal >> 16) == 0xffffu) {
          prod1 = false;
          rh1 = rt1;
        }
        if (!prod0 && !prod1) continue;
        // ---- load + 4x4 cull + d4 for both sub-tiles (hierarchy.py:190-199)
        const int j = pos + lane;
        Key dA = kInfKey, dB = kInfKey;
        uint32_t iA = kNoId, iB = kNoId;
#if STP_SID_PF
        const uint32_t cur_sid = pf_sid;
        if (j + 32 < k_total) pf_sid = __ldg(A.vals + start + j + 32);
#if STP_SID_PF > 1
        if (j + 32 < k_total) asm volatile("prefetch.global.L2 [%0];" ::"l"(A.recs + pf_sid));
#endif
#endif
        if (j < k_total) {
#if STP_SID_PF
          const uint32_t sid = cur_sid;
#else
          const uint32_t sid = A.vals[start + j];
#endif
          const SplatRec* r = A.recs + sid;
          double mx, my, a, b, ia, ic, thr, rect;
          ld256(&r->mx, mx, my, a, b);
          ld256(&r->inv_a, ia, ic, thr, rect);
          const double2 mxy = make_double2(mx, my);
          const double2 ab = make_double2(a, b);
          const double2 ct = make_double2(__ldg(&r->cc), thr);
          const double2 inv = make_double2(ia, ic);
          const float op = __ldg(&r->op);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            if (s ? !prod1 : !prod0) continue;
            const double r4x = (double)(sx0 + 4 * s);
            double ptx, pty;
            max_point(mxy.x, mxy.y, ab.x, ab.y, ct.x, inv.x, inv.y, r4x, r4y, 4.0, 0.25, ptx,
                      pty);
            if (alpha_keep(gpower(ab.x, ab.y, ct.x, ptx - mxy.x, pty - mxy.y), ct.y, op,
                           A.cfg.eps)) {
              const Key dv = dkey(key_rec_at(A.cam, *r, ptx, pty));
              if (s) {
                dB = dv;
                iB = sid;
              } else {
                dA = dv;
                iA = sid;
              }
            }
          }
        }
        STAT_ADD(0, j < k_total && prod0);
        STAT_ADD(0, j < k_total && prod1);
        STAT_ADD(1, iA != kNoId);
        STAT_ADD(1, iB != kNoId);
        pos += 32;
        const int nkA = __popc(__ballot_sync(kFull, iA != kNoId));
        const int nkB = __popc(__ballot_sync(kFull, iB != kNoId));
        PROF_ADD(0);
        STAT_ADD(2, lane == 0);
        STAT_ADD(3, lane == 0 && nkA + nkB > 0);
        if (nkA + nkB == 0) continue;
        // Sort the kept candidates by (d4, rank).  Common case (<= 16 kept per
        // sub-tile): compact each sub-tile's kept entries into one half-warp
        // and run ONE 16-wide bitonic network over both halves at once (10
        // stages, one array) instead of two 32-wide networks (15 stages, two
        // arrays).  Lane h*16+L then holds element L of sub-tile h.
        Key dS0, dS1;
        uint32_t iS0, iS1;
        int xS0, xS1;
        bool vS0, vS1;
        if (nkA <= 16 && nkB <= 16) {
          const unsigned bA = __ballot_sync(kFull, iA != kNoId);
          const unsigned bB = __ballot_sync(kFull, iB != kNoId);
          const int h = lane >> 4, L = lane & 15;
          const int nk = h ? nkB : nkA;
          const int src = select_bit32(h ? bB : bA, L < nk ? L : 0);
          const Key sdA = shfl_k(dA, src), sdB = shfl_k(dB, src);
          const uint32_t siA = __shfl_sync(kFull, iA, src), siB = __shfl_sync(kFull, iB, src);
          Key d = h ? sdB : sdA;
          uint32_t id = h ? siB : siA;
          if (L >= nk) {
            d = kInfKey;
            id = kNoId;
          }
#ifdef STP_WORK_STATS
          {  // sortedness of each half's candidates in bin order
            const Key pd = __shfl_up_sync(kFull, d, 1, 16);
            const uint32_t pi = __shfl_up_sync(kFull, id, 1, 16);
            const bool ok = L == 0 || L >= nk || lt(pd, pi, d, id);
            const unsigned bo = __ballot_sync(kFull, ok);
            STAT_ADD(12, L == 0 && nk > 1);
            STAT_ADD(13, L == 0 && nk > 1 && ((bo >> (lane & 16)) & 0xffffu) == 0xffffu);
          }
#endif
#if STP_RANK16
          // position of (d, id) among its half's candidates: 16 independent
          // shuffle + compare rounds instead of a 10-stage bitonic network
          // (the dependency chain, not the instruction count, was the cost)
          int rank = 0;
#pragma unroll kRankUnroll
          for (int jj = 0; jj < 16; ++jj) {
            const Key od = shfl_k(d, jj, 16);
            const uint32_t oi = __shfl_sync(kFull, id, jj, 16);
            rank += lt(od, oi, d, id);
          }
          dS0 = dS1 = d;
          iS0 = iS1 = id;
          xS0 = xS1 = rank;
#else
          half_sort16(d, id, L);
          dS0 = dS1 = d;
          iS0 = iS1 = id;
          xS0 = xS1 = L;
#endif
          vS0 = (h == 0) && L < nkA;
          vS1 = (h == 1) && L < nkB;
        } else {
          warp_sort2(dA, iA, dB, iB, lane);
          dS0 = dA;
          dS1 = dB;
          iS0 = iA;
          iS1 = iB;
          xS0 = xS1 = lane;
          vS0 = lane < nkA;
          vS1 = lane < nkB;
        }
        // ---- merge each sorted batch into its tail (heap_merge, :201), both
        // sub-tiles in the same instructions: every lane ranks its new
        // element(s) in its sub-tile's tail and the tails' elements in their
        // batches (lane-selected queues; sub-tiles without kept entries keep
        // their buffers).
        {
          const bool cpt = nkA <= 16 && nkB <= 16;
          // pass 1: element (s1, d1) of this lane -- the compact path's half
          // h, else sub-tile 0; pass 2 (non-compact only): sub-tile 1
          const int s1 = cpt ? (lane >> 4) : 0;
          const bool v1 = s1 ? vS1 : vS0;
          const Key d1 = s1 ? dS1 : dS0;
          const uint32_t i1 = s1 ? iS1 : iS0;
          const int x1 = s1 ? xS1 : xS0;
          const SubQ Q1 = subq(s1);
          if (v1) {
            Q1.bd()[x1] = d1;
            Q1.bi()[x1] = i1;
          }
          if (!cpt && vS1) {
            const SubQ Q = subq(1);
            Q.bd()[xS1] = dS1;
            Q.bi()[xS1] = iS1;
          }
          __syncwarp();
#ifdef STP_WORK_STATS
          {  // merges that are appends (every batch element after the tail)
            const int sl = lane & 1;
            const int nks = sl ? nkB : nkA, nts = sl ? nt1 : nt0, ths = sl ? th1 : th0;
            const SubQ Qs = subq(sl);
            const bool both = nks > 0 && nts > 0;
            bool app = false;
            if (lane < 2 && both) {
              const int cs = sl ? cur1 : cur0;
              app = lt(Qs.td(cs)[ths + nts - 1], Qs.ti(cs)[ths + nts - 1], Qs.bd()[0], Qs.bi()[0]);
            }
            STAT_ADD(14, lane < 2 && both);
            STAT_ADD(15, lane < 2 && app);
          }
#endif
          if (tail_inplace(qt)) {
            // qt == 64: tails hold <= 32 here, so every lane reads and ranks
            // at most one new element per sub-tile and two tail elements,
            // then all lanes write (single buffer)
            // Append fast path (65% of C3's merges, profiles/r2k): when the
            // batch's first element sorts after the tail's last, every new
            // element lands at nt + its batch index and the tail elements
            // keep their order -- no rank searches, and no moves at all if
            // the tail already starts at slot 0
            bool app0 = true, app1 = true;
            if (nkA && nt0) {
              const SubQ Q = subq(0);
              app0 = lt(Q.td(0)[th0 + nt0 - 1], Q.ti(0)[th0 + nt0 - 1], Q.bd()[0], Q.bi()[0]);
            }
            if (nkB && nt1) {
              const SubQ Q = subq(1);
              app1 = lt(Q.td(0)[th1 + nt1 - 1], Q.ti(0)[th1 + nt1 - 1], Q.bd()[0], Q.bi()[0]);
            }
            int rk1 = 0, rk2 = 0;
            if (v1)
              rk1 = (s1 ? app1 : app0)
                        ? (s1 ? nt1 : nt0)
                        : count_below(Q1.td(0) + (s1 ? th1 : th0), Q1.ti(0) + (s1 ? th1 : th0),
                                      s1 ? nt1 : nt0, d1, i1);
            if (!cpt && vS1) {
              const SubQ Q = subq(1);
              rk2 = app1 ? nt1 : count_below(Q.td(0) + th1, Q.ti(0) + th1, nt1, dS1, iS1);
            }
            // tail elements to (re)place: none for an append onto a tail at slot 0
            const int n0 = (nkA && !(app0 && th0 == 0)) ? nt0 : 0;
            const int n1 = (nkB && !(app1 && th1 == 0)) ? nt1 : 0;
            Key tv[2];
            uint32_t tiv[2];
            int trk[2], tpos[2], tst[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int u = lane + 32 * k;
              tst[k] = u >= n0;
              tpos[k] = -1;
              if (u < n0 + n1) {
                const int st = tst[k];
                const int t = u - (st ? n0 : 0);
                const SubQ Q = subq(st);
                const int th = st ? th1 : th0;
                tv[k] = Q.td(0)[th + t];
                tiv[k] = Q.ti(0)[th + t];
                trk[k] = (st ? app1 : app0) ? 0
                                            : count_below(Q.bd(), Q.bi(), st ? nkB : nkA, tv[k],
                                                          tiv[k]);
                tpos[k] = t;
              }
            }
            __syncwarp();
            if (v1) {
              Q1.td(0)[x1 + rk1] = d1;
              Q1.ti(0)[x1 + rk1] = i1;
            }
            if (!cpt && vS1) {
              const SubQ Q = subq(1);
              Q.td(0)[xS1 + rk2] = dS1;
              Q.ti(0)[xS1 + rk2] = iS1;
            }
#pragma unroll
            for (int k = 0; k < 2; ++k)
              if (tpos[k] >= 0) {
                const SubQ Q = subq(tst[k]);
                Q.td(0)[tpos[k] + trk[k]] = tv[k];
                Q.ti(0)[tpos[k] + trk[k]] = tiv[k];
              }
            __syncwarp();
            if (nkA) {
              th0 = 0;
              nt0 += nkA;
            }
            if (nkB) {
              th1 = 0;
              nt1 += nkB;
            }
            PROF_ADD(1);
            continue;
          }
          if (v1) {
            const int cur = s1 ? cur1 : cur0, th = s1 ? th1 : th0, nt = s1 ? nt1 : nt0;
            const int rk = count_below(Q1.td(cur) + th, Q1.ti(cur) + th, nt, d1, i1);
            Q1.td(cur ^ 1)[x1 + rk] = d1;
            Q1.ti(cur ^ 1)[x1 + rk] = i1;
          }
          if (!cpt && vS1) {
            const SubQ Q = subq(1);
            const int rk = count_below(Q.td(cur1) + th1, Q.ti(cur1) + th1, nt1, dS1, iS1);
            Q.td(cur1 ^ 1)[xS1 + rk] = dS1;
            Q.ti(cur1 ^ 1)[xS1 + rk] = iS1;
          }
          // the tails' elements, both sub-tiles in one index space
          const int n0 = nkA ? nt0 : 0, n1 = nkB ? nt1 : 0;
          for (int u = lane; u < n0 + n1; u += 32) {
            const int st = u >= n0;
            const int t = u - (st ? n0 : 0);
            const SubQ Q = subq(st);
            const int cur = st ? cur1 : cur0, th = st ? th1 : th0;
            const Key tv = Q.td(cur)[th + t];
            const uint32_t tiv = Q.ti(cur)[th + t];
            const int rk = count_below(Q.bd(), Q.bi(), st ? nkB : nkA, tv, tiv);
            Q.td(cur ^ 1)[t + rk] = tv;
            Q.ti(cur ^ 1)[t + rk] = tiv;
          }
          __syncwarp();
          if (nkA) {
            cur0 ^= 1;
            th0 = 0;
            nt0 += nkA;
          }
          if (nkB) {
            cur1 ^= 1;
            th1 = 0;
            nt1 += nkB;
          }
        }
        PROF_ADD(1);
        continue;
      }
      // ---- end of the bin, tails empty: flush a sub-tile's mid queues
      {
        const int fs = prod0 ? 0 : 1;
        const SubQ Q = subq(fs);
        const int nm = fs ? nm1 : nm0, rt = fs ? rt1 : rt0;
        const uint32_t* mi = Q.i + Q.o_mid(mq);
        uint32_t* ring = Q.ring(mq, R);
        for (int sl = lane & 7; sl < nm; sl += 8) ring[(rt + sl) & (R - 1)] = mi[sl];
        __syncwarp();
        if (fs) {
          rt1 += nm;
          nm1 = 0;
          prod1 = false;
        } else {
          rt0 += nm;
          nm0 = 0;
          prod0 = false;
        }
      }
    }
    // heads drain in ascending (t, rank) (hierarchy.py:215-217); no-ops for
    // terminated sub-tiles
#pragma unroll
    for (int i = 0; i < QH; ++i)
      if (i < H.n) blend<XM>(P, A, kdbl(H.t[i]), H.a[i], H.id[i]);
    PROF_ADD(4);

    xm_done<XM>(P, A);
    if (P.pix >= 0 && XM != XM_BWD) {
      const float T = (float)P.T;
      const float c0 = P.C0 + (float)(P.T * A.cfg.bg[0]);
      const float c1 = P.C1 + (float)(P.T * A.cfg.bg[1]);
      const float c2 = P.C2 + (float)(P.T * A.cfg.bg[2]);
      A.out.color[P.pix * 3 + 0] = c0;
      A.out.color[P.pix * 3 + 1] = c1;
      A.out.color[P.pix * 3 + 2] = c2;
      A.out.transmittance[P.pix] = T;
      if (A.out.depth) A.out.depth[P.pix] = P.D;
      if (A.cfg.rec_cap > 0) A.out.rec_count[P.pix] = P.rc;
      if (!(isfinite(c0) && isfinite(c1) && isfinite(c2) && isfinite(T)))
        atomicAdd(A.counters + C_NONFINITE, 1ull);
    }
  }
}

#ifndef STP_SMEM_PAD
#define STP_SMEM_PAD 0  // experiments: extra shared memory per block (less L1)
#endif
size_t render_smem_bytes(int qt, int qm) {
  return kWarpsPerBlock * warp_smem_bytes(qt, qm) + STP_SMEM_PAD;
}

#ifndef STP_K6_BPS
#define STP_K6_BPS 0  // cap on resident K6 blocks per SM (0: the occupancy maximum)
#endif

template <int QH, bool EXACT, int QMX, int QT = 0, int XM = XM_NONE>
static void launch_render_t(const RenderArgs& A, size_t smem, cudaStream_t s) {
  static size_t attr = 0;
  static int blocks_per_sm = 0, n_sm = 0;
  if (smem != attr || blocks_per_sm == 0) {
    cudaFuncSetAttribute(k_render<QH, EXACT, QMX, QT, XM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = smem;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_render<QH, EXACT, QMX, QT, XM>,
                                                  kRenderThreads, smem);
    n_sm = device_sm_count();
    if (STP_K6_BPS > 0 && blocks_per_sm > STP_K6_BPS) blocks_per_sm = STP_K6_BPS;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int want = (A.n_items * 8 + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int grid = min(want, n_sm * blocks_per_sm);
  if (grid > 0) k_render<QH, EXACT, QMX, QT, XM><<<grid, kRenderThreads, smem, s>>>(A);
}

// ---------------------------------------------------------------------------
// K6 under GlobalZ (rasterizer.py:472-485): every pixel blends the bin in its
// sorted (view z, rank) order -- the 3DGS baseline the paper compares with.
// _TileCtx.alphas (:412-422: alpha capped, zeroed below eps) and
// _blend_ordered (:432-459: T_k = prod(1 - alpha_i), an entry blends while the
// T before it is >= termination, final T = the first value below); the depth
// output blends the distance to the Gaussian's mean (:478-482).  One block of
// 256 threads per 16x16 tile, one thread per pixel; the bin streams through
// shared memory 256 entries at a time and the block stops when every pixel
// has terminated.
constexpr int kGzThreads = 256;

struct GzArgs {
  int xm;          // XM_* (runtime: the GlobalZ kernel is not register bound)
  int tile0;       // first tile of the band; n_tiles = band length
  DevGrads grad;
  const SplatRec* __restrict__ recs;
  const uint32_t* __restrict__ vals;
  const uint2* __restrict__ ranges;
  const double2* __restrict__ aux;  // (view z, |mean - origin|)
  DevCam cam;
  DevCfg cfg;
  int gw, n_tiles;
  StpOutputs out;
  unsigned long long* counters;
  const double* col64;
};

__global__ void __launch_bounds__(kGzThreads) k_render_globalz(GzArgs A) {
  __shared__ double s_tab[64];
  __shared__ double s_mx[kGzThreads], s_my[kGzThreads], s_a[kGzThreads], s_b[kGzThreads],
      s_c[kGzThreads], s_dist[kGzThreads];
  __shared__ float4 s_oc[kGzThreads];  // opacity, colour
  __shared__ uint32_t s_id[kGzThreads];
#if STP_WIN_STRIP
  __shared__ double s_ia[kGzThreads], s_thr[kGzThreads];
  __shared__ unsigned s_msk[kGzThreads / 32][kGzThreads / 32];  // [warp][32-entry group]
#endif
  const int tid = threadIdx.x;
  if (tid < 64) s_tab[tid] = kExp2Tab[tid];
  // the per-blend helpers take RenderArgs
  RenderArgs R;
  R.recs = A.recs;
  R.cam = A.cam;
  R.cfg = A.cfg;
  R.out = A.out;
  R.counters = A.counters;
  R.grad = A.grad;
  R.col64 = A.col64;
  const bool need_t = A.cfg.rec_cap > 0 || A.xm == XM_SERR ||
                      (A.xm == XM_F64 && A.out.sort_error != nullptr);
  for (int band = blockIdx.x; band < A.n_tiles; band += gridDim.x) {
    const int tile = band + A.tile0;
    const int tx = tile % A.gw, ty = tile / A.gw;
    const int gx = tx * kTile + (tid & 15), gy = ty * kTile + (tid >> 4);
    const bool in_img = gx < A.cam.W && gy < A.cam.H;
    Pixel P;
    P.pix = in_img ? (int64_t)gy * A.cam.W + gx : -1;
    P.px = (double)gx + 0.5;
    P.py = (double)gy + 0.5;
    P.u = P.w = P.vn = 0.0;
    if (need_t) cam_ray(A.cam, P.px, P.py, P.u, P.w, P.vn);
    P.T = in_img ? 1.0 : 0.0;
    P.C0 = P.C1 = P.C2 = P.D = 0.f;
    P.rc = 0;
    switch (A.xm) {
      case XM_BWD: xm_init<XM_BWD>(P, R); break;
      default: xm_init<XM_NONE>(P, R); break;
    }
    const uint2 rg = A.ranges[tile];
    for (uint32_t base = rg.x; base < rg.y; base += kGzThreads) {
      // all pixels terminated: the rest of the bin blends nothing
      if (__syncthreads_count(P.T >= A.cfg.term) == 0) break;
      const uint32_t j = base + tid;
      if (j < rg.y) {
        const uint32_t id = A.vals[j];
        const SplatRec* r = A.recs + id;
        double mx, my, a, b;
        ld256(&r->mx, mx, my, a, b);
        s_mx[tid] = mx;
        s_my[tid] = my;
        s_a[tid] = a;
        s_b[tid] = b;
        s_c[tid] = __ldg(&r->cc);
        s_oc[tid] = __ldg(reinterpret_cast<const float4*>(&r->op));
        s_dist[tid] = A.aux[id].y;
        s_id[tid] = id;
#if STP_WIN_STRIP
        s_ia[tid] = __ldg(&r->inv_a);
        s_thr[tid] = __ldg(&r->thr);
#endif
      }
      __syncthreads();
      const int n = (int)min((uint32_t)kGzThreads, rg.y - base);
#if STP_WIN_STRIP
      // warp-level strip cull (the warp's pixels are a 16 x 2 strip): lane l
      // tests staged entries l, l + 32, ...; the warp walks the survivors in
      // bin order (strip_may_pass's bound, on the staged fields)
      unsigned* const msk = s_msk[tid >> 5];
      {
        const int lane = tid & 31;
        const double sx = (double)(tx * kTile), sy = (double)(ty * kTile + 2 * (tid >> 5));
#pragma unroll
        for (int q = 0; q < kGzThreads / 32; ++q) {
          const int k = 32 * q + lane;
          bool keep = k < n;
          if (keep && A.cfg.eps > 0.0) {
            const double a = s_a[k], b = s_b[k], c = s_c[k], ia = s_ia[k], thr = s_thr[k];
            if (a > 0.0) {
              const double X0 = sx + 0.5 - s_mx[k], X1 = sx + 15.5 - s_mx[k];
              double qmin = INFINITY, mag = 0.0;
#pragma unroll
              for (int row = 0; row < 2; ++row) {
                const double dy = sy + 0.5 + row - s_my[k];
                const double dx = fmin(fmax(-b * dy * ia, X0), X1);
                const double t1 = 0.5 * a * dx * dx, t2 = b * dx * dy, t3 = 0.5 * c * dy * dy;
                qmin = fmin(qmin, t1 + t2 + t3);
                mag = fmax(mag, fabs(t1) + fabs(t2) + fabs(t3));
              }
              keep = !(qmin > thr + 1e-6 * (1.0 + fabs(thr)) + 1e-9 * mag);
            }
          }
          const unsigned bq = __ballot_sync(kFull, keep);
          if (lane == 0) msk[q] = bq;
        }
        __syncwarp();
      }
      for (int q = 0; q < kGzThreads / 32; ++q)
      for (unsigned mq = msk[q]; mq; mq &= mq - 1) {
        const int k = 32 * q + __ffs(mq) - 1;
        if (!(P.T >= A.cfg.term)) continue;
#else
      for (int k = 0; k < n && P.T >= A.cfg.term; ++k) {
#endif
        const double dx = P.px - s_mx[k], dy = P.py - s_my[k];
        const double pw = gpower(s_a[k], s_b[k], s_c[k], dx, dy);
        const float4 oc = s_oc[k];
        double al = (double)oc.x * exp_neg_nb(min_le(pw, 700.0), s_tab);
        al = min_le(al, A.cfg.cap);
        if (al < A.cfg.eps) continue;  // alpha 0: no weight, T unchanged
        const double wt = al * P.T;
        const float wf = (float)wt;
        P.C0 += oc.y * wf;
        P.C1 += oc.z * wf;
        P.C2 += oc.w * wf;
        P.D += (float)(s_dist[k] * wt);
        if (A.xm == XM_F64) P.dd += s_dist[k] * wt;
        double t = 0.0;
        if (need_t) {
          const SplatRec* r = A.recs + s_id[k];
          t = key_rec(r->m, r->q0, r->q1, r->q2, P.u, P.w, P.vn);
          if (A.cfg.rec_cap > 0) write_record(A.out, A.cfg.rec_cap, P.pix, P.rc++, t, al, s_id[k]);
        }
        switch (A.xm) {
          case XM_SERR: xm_step<XM_SERR>(P, R, t, al, s_id[k], oc); break;
          case XM_FWD: xm_step<XM_FWD>(P, R, t, al, s_id[k], oc); break;
          case XM_BWD: xm_step<XM_BWD>(P, R, t, al, s_id[k], oc); break;
          case XM_F64: xm_step<XM_F64>(P, R, t, al, s_id[k], oc); break;
          default: break;
        }
        P.T = P.T * (1.0 - al);
      }
      __syncthreads();
    }
    switch (A.xm) {
      case XM_SERR: xm_done<XM_SERR>(P, R); break;
      case XM_FWD: xm_done<XM_FWD>(P, R); break;
      case XM_F64: xm_done<XM_F64>(P, R); break;
      default: break;
    }
    if (P.pix >= 0 && A.xm != XM_BWD) {
      const float Tf = (float)P.T;
      const float c0 = P.C0 + (float)(P.T * A.cfg.bg[0]);
      const float c1 = P.C1 + (float)(P.T * A.cfg.bg[1]);
      const float c2 = P.C2 + (float)(P.T * A.cfg.bg[2]);
      A.out.color[P.pix * 3 + 0] = c0;
      A.out.color[P.pix * 3 + 1] = c1;
      A.out.color[P.pix * 3 + 2] = c2;
      A.out.transmittance[P.pix] = Tf;
      if (A.out.depth) A.out.depth[P.pix] = P.D;
      if (A.cfg.rec_cap > 0) A.out.rec_count[P.pix] = P.rc;
      if (!(isfinite(c0) && isfinite(c1) && isfinite(c2) && isfinite(Tf)))
        atomicAdd(A.counters + C_NONFINITE, 1ull);
    }
    __syncthreads();
  }
}

static void launch_render_globalz(const Frame& f, const StpOutputs& out, cudaStream_t s, int xm,
                                  const DevGrads* g) {
  GzArgs A;
  A.xm = xm;
  if (g) A.grad = *g;
  A.recs = f.recs;
  A.vals = f.vals;
  A.ranges = f.ranges;
  A.aux = f.aux;
  A.cam = f.cam;
  A.cfg = f.cfg;
  A.gw = f.gw;
  A.tile0 = f.tile0;
  A.n_tiles = f.tile1 - f.tile0;
  A.out = out;
  A.counters = f.counters;
  A.col64 = f.col64;
  if (A.n_tiles > 0) k_render_globalz<<<A.n_tiles, kGzThreads, 0, s>>>(A);
}

// ---------------------------------------------------------------------------
// K6 under Window(size) (rasterizer.py:504-588) and FullPerPixel (:488-501).
// The bins are the hierarchical ones (per-tile t_opt keys, exact culling).
// One warp per block = 32 pixels (a 16 x 2 strip of a tile, 8 warps per
// tile, warps independent: a warp stops when its pixels have terminated);
// every entry is evaluated exactly as the hierarchical pixel stage does
// (alpha, eps test, cap, pixel-ray t_opt).  Window: the window is a
// per-pixel binary min-heap of (t, rank) in shared memory, laid out
// [slot][lane] so every heap access of a warp is bank-conflict free.  The
// reference's window is a set with "emit the smaller of (incoming, window
// minimum) on overflow, drain in (t, rank) order" -- exactly a bounded
// min-heap (ranks are unique, so the order is total).  A slot stores (t,
// rank) only; alpha of a popped entry is re-evaluated (emit_eval_bf is
// deterministic: the same t and alpha as at insertion), which keeps 12 B per
// slot: up to kWindowMax entries per pixel.  (Round 1 kept windows up to 16
// in registers, one thread per pixel in 256-thread tile blocks: measured
// slower at every size, C3 K6 Window(3) 5.4 vs 3.9 ms, (8) 5.4 vs 4.8,
// (16) 14.8 vs 5.6 -- profiles/r2i -- and removed.)
constexpr int kWindowMax = STP_WINDOW_MAX;
constexpr int kWinPix = 32;

__host__ __device__ inline size_t window_smem_bytes(int cap) {
  return (size_t)cap * kWinPix * (sizeof(double) + sizeof(uint32_t));
}

// FullPerPixel (rasterizer.py:488-501) on the same kernel (FULL): the exact
// per-pixel order by repeated top-K selection with a K-slot MAX-heap -- a
// pass over the bin keeps the K smallest valid (t, rank) above the last
// blended one, heap-sorts them ascending and blends them; the next pass
// continues above the K-th.  A pixel is done when a pass keeps fewer than K
// or it terminates.  C3 K6 (profiles/r2i): K = 16 in registers 112.9 ms,
// heap K = 16 61.1 ms, 24 52.0, 32 47.9, 48 46.8, 64 53.1, 128 64.4 (fewer
// passes vs occupancy).
#ifndef STP_FULL_HEAP
#define STP_FULL_HEAP 48  // K (round 1: K = 16 selection in registers, 112.9 ms)
#endif

// Strip cull of the Window / FullPerPixel scans: may entry `id` reach
// alpha >= eps at any pixel centre of the 16 x 2 strip with top-left pixel
// (x0, y0)?  Exact minimum of the power over each row's segment of centres
// (a 1-D quadratic, vertex clamped to the segment) against thr = log(op/eps)
// plus a margin, so a culled entry fails the float64 alpha test at every
// pixel of the strip (NaN fields are kept: the exact test decides them).
__device__ __forceinline__ bool strip_may_pass(const SplatRec* r, double x0, double y0) {
  double mx, my, a, b, ia, ic, thr, rect;
  ld256(&r->mx, mx, my, a, b);
  ld256(&r->inv_a, ia, ic, thr, rect);
  const double c = __ldg(&r->cc);
  if (!(a > 0.0)) return true;  // not convex in x (e.g. a SplatBatch conic): no bound
  const double X0 = x0 + 0.5 - mx, X1 = x0 + 15.5 - mx;
  double qmin = INFINITY, mag = 0.0;
#pragma unroll
  for (int row = 0; row < 2; ++row) {
    const double dy = y0 + 0.5 + row - my;
    const double dx = fmin(fmax(-b * dy * ia, X0), X1);  // vertex of 0.5 a dx^2 + b dy dx
    const double t1 = 0.5 * a * dx * dx, t2 = b * dx * dy, t3 = 0.5 * c * dy * dy;
    qmin = fmin(qmin, t1 + t2 + t3);
    mag = fmax(mag, fabs(t1) + fabs(t2) + fabs(t3));
  }
  return !(qmin > thr + 1e-6 * (1.0 + fabs(thr)) + 1e-9 * mag);
}

template <int XM, bool FULL>
__global__ void __launch_bounds__(kWinPix) k_render_window(RenderArgs A, int cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_tab[64];
  for (int i = threadIdx.x; i < 64; i += kWinPix) s_tab[i] = kExp2Tab[i];
  __syncwarp();
  const int lane = threadIdx.x;
  double* hd = reinterpret_cast<double*>(smem_raw) + lane;                    // [slot][lane]
  uint32_t* hid = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(smem_raw) +
                                              (size_t)cap * kWinPix) + lane;
  const double term = A.cfg.term;
  // heap order: "a belongs nearer the root than b" -- min-heap (Window) or
  // max-heap (FULL's top-K selection)
  auto before = [](double ad, uint32_t ai, double bd, uint32_t bi) {
    return FULL ? lt(bd, bi, ad, ai) : lt(ad, ai, bd, bi);
  };
  for (int item = blockIdx.x; item < A.n_items * 8; item += gridDim.x) {
    const int tile = item / 8 + A.tile0, strip = item % 8;
    const int tx = tile % A.gw, ty = tile / A.gw;
    Pixel P;
    {
      const int gx = tx * kTile + (lane & 15), gy = ty * kTile + 2 * strip + (lane >> 4);
      const bool in_img = gx < A.cam.W && gy < A.cam.H;
      P.pix = in_img ? (int64_t)gy * A.cam.W + gx : -1;
      P.px = (double)gx + 0.5;
      P.py = (double)gy + 0.5;
      cam_ray(A.cam, P.px, P.py, P.u, P.w, P.vn);
      P.T = in_img ? 1.0 : 0.0;
      P.C0 = P.C1 = P.C2 = P.D = 0.f;
      P.rc = 0;
      xm_init<XM>(P, A);
    }
    const double sx = (double)(tx * kTile), sy = (double)(ty * kTile + 2 * strip);
    const bool strip_ok = A.cfg.eps > 0.0;  // eps <= 0: every entry passes alpha
    // place (xd, xi) in the root's hole and sift it down over n elements
    auto sift_down = [&](double xd, uint32_t xi, int n) {
      int p = 0;
      for (;;) {
        int c = 2 * p + 1;
        if (c >= n) break;
        double cd = hd[(size_t)c * kWinPix];
        uint32_t ci = hid[(size_t)c * kWinPix];
        if (c + 1 < n) {
          const double rd = hd[(size_t)(c + 1) * kWinPix];
          const uint32_t ri = hid[(size_t)(c + 1) * kWinPix];
          if (before(rd, ri, cd, ci)) {
            ++c;
            cd = rd;
            ci = ri;
          }
        }
        if (!before(cd, ci, xd, xi)) break;
        hd[(size_t)p * kWinPix] = cd;
        hid[(size_t)p * kWinPix] = ci;
        p = c;
      }
      hd[(size_t)p * kWinPix] = xd;
      hid[(size_t)p * kWinPix] = xi;
    };
    auto sift_up = [&](double xd, uint32_t xi, int c) {
      while (c > 0) {
        const int p = (c - 1) >> 1;
        const double pd = hd[(size_t)p * kWinPix];
        const uint32_t pi = hid[(size_t)p * kWinPix];
        if (!before(xd, xi, pd, pi)) break;
        hd[(size_t)c * kWinPix] = pd;
        hid[(size_t)c * kWinPix] = pi;
        c = p;
      }
      hd[(size_t)c * kWinPix] = xd;
      hid[(size_t)c * kWinPix] = xi;
    };
    // blend (t0, i0): alpha re-evaluated (deterministic: the value at insertion)
    auto blend_at = [&](double t0, uint32_t i0) {
      double t, al;
      emit_eval_bf(P, A, i0, s_tab, t, al);
      blend<XM>(P, A, t0, al, i0);
    };
    const uint2 rg = A.ranges[tile];
    if (!FULL) {
      int n = 0;
      bool stop = false;
      for (uint32_t j0 = rg.x; j0 < rg.y && !stop; j0 += 32) {
        // lane-per-entry strip cull, then the survivors in bin order
        const uint32_t jl = j0 + lane;
        const uint32_t idl = jl < rg.y ? A.vals[jl] : 0u;
        unsigned surv = __ballot_sync(kFull, jl < rg.y && (!STP_WIN_STRIP || !strip_ok ||
                                                          strip_may_pass(A.recs + idl, sx, sy)));
        while (surv) {
          const int src = __ffs(surv) - 1;
          surv &= surv - 1;
          if (!__any_sync(kFull, P.T >= term)) {
            stop = true;
            break;
          }
          const uint32_t id = __shfl_sync(kFull, idl, src);
          double t, al;
          const bool pass = emit_eval_pre(P, A, id, s_tab, t, al);
          if (!(pass && P.T >= term)) continue;
          if (n < cap) {
            sift_up(t, id, n++);
          } else if (lt(t, id, hd[0], hid[0])) {
            blend<XM>(P, A, t, al, id);  // the incoming entry is the smallest: emitted
          } else {
            // emit the minimum; the incoming entry takes its place
            const double t0 = hd[0];
            const uint32_t i0 = hid[0];
            sift_down(t, id, n);
            blend_at(t0, i0);
          }
        }
      }
      // drain in ascending (t, rank) (rasterizer.py:565-573); no-ops once terminated
      while (n > 0 && P.T >= term) {
        const double t0 = hd[0];
        const uint32_t i0 = hid[0];
        --n;
        sift_down(hd[(size_t)n * kWinPix], hid[(size_t)n * kWinPix], n);
        blend_at(t0, i0);
      }
    } else {
      double lo_t = -INFINITY;
      uint32_t lo_id = 0;
      bool first = true, more = true;
      while (__any_sync(kFull, more && P.T >= term)) {
        // every lane runs the scan (lane-per-entry cull, warp shuffles);
        // only the pixels still selecting (act) evaluate and keep entries
        const bool act = more && P.T >= term;
        int n = 0;
        for (uint32_t j0 = rg.x; j0 < rg.y; j0 += 32) {
          const uint32_t jl = j0 + lane;
          const uint32_t idl = jl < rg.y ? A.vals[jl] : 0u;
          unsigned surv = __ballot_sync(kFull, jl < rg.y && (!STP_WIN_STRIP || !strip_ok ||
                                                            strip_may_pass(A.recs + idl, sx, sy)));
          while (surv) {
            const int src = __ffs(surv) - 1;
            surv &= surv - 1;
            const uint32_t id = __shfl_sync(kFull, idl, src);
            if (!act) continue;
            double t, al;
            if (!emit_eval_pre(P, A, id, s_tab, t, al)) continue;
            if (!first && !lt(lo_t, lo_id, t, id)) continue;  // blended by an earlier pass
            if (n < cap) sift_up(t, id, n++);
            else if (lt(t, id, hd[0], hid[0])) sift_down(t, id, n);  // replaces the maximum
          }
        }
        if (!act) continue;
        // heap-sort ascending in place, then blend in order
        for (int m = n - 1; m > 0; --m) {
          const double xd = hd[(size_t)m * kWinPix];
          const uint32_t xi = hid[(size_t)m * kWinPix];
          hd[(size_t)m * kWinPix] = hd[0];
          hid[(size_t)m * kWinPix] = hid[0];
          sift_down(xd, xi, m);
        }
        for (int i = 0; i < n && P.T >= term; ++i)
          blend_at(hd[(size_t)i * kWinPix], hid[(size_t)i * kWinPix]);
        if (n < cap) more = false;
        else {
          lo_t = hd[(size_t)(n - 1) * kWinPix];
          lo_id = hid[(size_t)(n - 1) * kWinPix];
        }
        first = false;
      }
    }
    xm_done<XM>(P, A);
    if (P.pix >= 0 && XM != XM_BWD) {
      const float T = (float)P.T;
      const float c0 = P.C0 + (float)(P.T * A.cfg.bg[0]);
      const float c1 = P.C1 + (float)(P.T * A.cfg.bg[1]);
      const float c2 = P.C2 + (float)(P.T * A.cfg.bg[2]);
      A.out.color[P.pix * 3 + 0] = c0;
      A.out.color[P.pix * 3 + 1] = c1;
      A.out.color[P.pix * 3 + 2] = c2;
      A.out.transmittance[P.pix] = T;
      if (A.out.depth) A.out.depth[P.pix] = P.D;
      if (A.cfg.rec_cap > 0) A.out.rec_count[P.pix] = P.rc;
      if (!(isfinite(c0) && isfinite(c1) && isfinite(c2) && isfinite(T)))
        atomicAdd(A.counters + C_NONFINITE, 1ull);
    }
  }
}

template <int XM, bool FULL>
static void launch_window_t(const RenderArgs& A, int cap, cudaStream_t s) {
  const size_t smem = window_smem_bytes(cap);
  cudaFuncSetAttribute(k_render_window<XM, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_window<XM, FULL>, kWinPix,
                                                smem);
  const long long items = (long long)A.n_items * 8;
  const long long grid = std::min<long long>(items, (long long)device_sm_count() *
                                                        std::max(per_sm, 1));
  k_render_window<XM, FULL><<<(int)grid, kWinPix, smem, s>>>(A, cap);
}

template <bool FULL>
static void launch_window_xm(const RenderArgs& A, int cap, int xm, cudaStream_t s) {
  switch (xm) {
    case XM_SERR: launch_window_t<XM_SERR, FULL>(A, cap, s); break;
    case XM_FWD: launch_window_t<XM_FWD, FULL>(A, cap, s); break;
    case XM_BWD: launch_window_t<XM_BWD, FULL>(A, cap, s); break;
    case XM_F64: launch_window_t<XM_F64, FULL>(A, cap, s); break;
    default: launch_window_t<XM_NONE, FULL>(A, cap, s); break;
  }
}

static void launch_render_pixelsort(const Frame& f, const RenderArgs& A, int xm,
                                    cudaStream_t s) {
  if (A.n_items <= 0) return;
  if (f.sort_mode == STP_MODE_FULL) launch_window_xm<true>(A, STP_FULL_HEAP, xm, s);
  else launch_window_xm<false>(A, f.cfg.q_head, xm, s);
}

// K6 dispatch.  xm: XM_NONE (render), or with `g` the backward replays
// XM_FWD / XM_BWD; a non-null out.sort_error selects XM_SERR.
void launch_render(const Frame& f, int buf, const StpOutputs& out, cudaStream_t s, int xm,
                   const DevGrads* g) {
  if (xm == XM_NONE && out.color64) xm = XM_F64;
  if (xm == XM_NONE && out.sort_error) xm = XM_SERR;
  if (f.globalz) {
    launch_render_globalz(f, out, s, xm, g);
    return;
  }
  RenderArgs A;
  A.recs = f.recs;
  A.log_eps = (float)log(f.cfg.eps);
  A.vals = f.vals;
  A.ranges = f.ranges;
  A.cam = f.cam;
  A.cfg = f.cfg;
  A.gw = f.gw;
  A.tile0 = f.tile0;
  A.n_items = f.tile1 - f.tile0;
  A.out = out;
  A.counters = f.counters;
  A.col64 = f.col64;
  if (g) A.grad = *g;
  if (f.sort_mode == STP_MODE_FULL || f.sort_mode == STP_MODE_WINDOW) {
    launch_render_pixelsort(f, A, xm, s);
    return;
  }
  const size_t smem = render_smem_bytes(f.cfg.q_tail, f.cfg.q_mid);
  if (xm != XM_NONE) {
    // diagnostics / backward: the default queues or the generic kernel
    const bool dflt = f.cfg.q_tail == 64 && f.cfg.q_mid == 8 && f.cfg.q_head == 4;
    switch (xm) {
      case XM_SERR:
        if (dflt) launch_render_t<4, true, 8, 64, XM_SERR>(A, smem, s);
        else launch_render_t<16, false, 0, 0, XM_SERR>(A, smem, s);
        break;
      case XM_FWD:
        if (dflt) launch_render_t<4, true, 8, 64, XM_FWD>(A, smem, s);
        else launch_render_t<16, false, 0, 0, XM_FWD>(A, smem, s);
        break;
      case XM_F64:
        if (dflt) launch_render_t<4, true, 8, 64, XM_F64>(A, smem, s);
        else launch_render_t<16, false, 0, 0, XM_F64>(A, smem, s);
        break;
      default:
        if (dflt) launch_render_t<4, true, 8, 64, XM_BWD>(A, smem, s);
        else launch_render_t<16, false, 0, 0, XM_BWD>(A, smem, s);
        break;
    }
    return;
  }
  if (f.cfg.q_mid > 8) {
    launch_render_t<16, false, 0>(A, smem, s);
    return;
  }
  switch (f.cfg.q_head) {
    case 1: launch_render_t<1, true, 8>(A, smem, s); break;
    case 2: launch_render_t<2, true, 8>(A, smem, s); break;
    case 4:
      if (STP_QT_SPECIALIZE && f.cfg.q_tail == 64 && f.cfg.q_mid == 8)
        launch_render_t<4, true, 8, 64>(A, smem, s);
      else launch_render_t<4, true, 8>(A, smem, s);
      break;
    case 8: launch_render_t<8, true, 8>(A, smem, s); break;
    case 16: launch_render_t<16, true, 8>(A, smem, s); break;
    default: launch_render_t<16, false, 8>(A, smem, s); break;
  }
}

}  // namespace stp
