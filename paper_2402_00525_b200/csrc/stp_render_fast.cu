// K6 fast path: hierarchy.render_tile (hierarchy.py:27-219) in fp32 with
// certified decisions.
//
// Same work decomposition and queue pipeline as the float64 kernel
// (stp_render.cu: one warp per horizontally adjacent pair of 4x4 sub-tiles,
// per-SM tile scheduling, tail / mid queues and emit rings in shared memory,
// register head queues).  What changes is the number format of the state:
//
//  * every key (4x4 d4, 2x2 d2, pixel t) is EVALUATED in float64 (camera-
//    space form, SplatRec32) but STORED, shuffled and compared as fp32.  A
//    stored key is within 2^-23 relative of the reference's float64 value,
//    so a comparison whose operands differ by more than that window is the
//    reference's comparison; inside the window (~1 in 10^5 comparisons) both
//    keys are recomputed with the reference's float64 formula and compared
//    with the rank tie-break (exact_less).  Every sort, merge, pop and
//    insertion therefore takes the reference's order (hierarchy.py:110,163,203);
//  * the 4x4 cull and the pixel eps test are decided in float64 (as in the
//    exact kernel); alpha itself is fp32 (MUFU ex2) with a relative error
//    bound;
//  * transmittance is fp32 with a running relative error bound; a
//    termination test (hierarchy.py:82-84, 187-189) that the bound cannot
//    decide aborts the sub-tile pair, which the float64 kernel (stp_render.cu,
//    list mode) then renders.
//
// So the blend sequence of every pixel equals the exact kernel's; colour,
// depth and transmittance differ only by fp32 rounding of the weights.
#include "stp_common.cuh"

namespace stp {

#ifndef STP_FAST_MINB
#define STP_FAST_MINB 4
#endif
constexpr int kFWarpsPerBlock = 4;
constexpr int kFThreads = 32 * kFWarpsPerBlock;
constexpr unsigned kNoIdF = 0xffffffffu;
constexpr float kU = 0x1p-24f;         // fp32 unit roundoff

// Keys are fp32 values stored as order-preserving int32 ("key index"): the
// float64 key rounded to nearest fp32, then the sign-magnitude bits flipped
// so that signed integer order is float order.  The reference's float64 key
// lies strictly between the neighbouring fp32 values of a stored key (half
// an ulp of rounding + a float64 formula difference << ulp), so two stored
// keys whose indices differ by >= 2 are ordered like the reference's keys;
// indices within 1 are settled in float64 (exact_less).
typedef int32_t Key;
constexpr Key kPad = 0x7fffffff;   // empty slot: above every real key (NaN bits)

__device__ __forceinline__ Key f2key(float f) {
  const int32_t b = __float_as_int(f);
  return b ^ ((b >> 31) & 0x7fffffff);
}
__device__ __forceinline__ float key2f(Key k) { return __int_as_float(k ^ ((k >> 31) & 0x7fffffff)); }

#ifdef STP_PHASE_PROF
#define FSTAT(slot, pred)                                                             \
  do {                                                                                \
    const unsigned _b = __ballot_sync(kFull, (pred));                                 \
    if (lane == 0 && _b) atomicAdd(A.counters + C_STAT + (slot), (unsigned long long)__popc(_b)); \
  } while (0)
#else
#define FSTAT(slot, pred) (void)0
#endif

struct FastArgs {
  const SplatRec* __restrict__ recs;     // float64 records (cull, exact paths)
  const SplatRec32* __restrict__ r32;    // fp32 records
  const uint32_t* __restrict__ vals;
  const uint2* __restrict__ ranges;
  const DevCam* __restrict__ camp;       // the camera in global memory (exact paths)
  DevCam cam;
  DevCfg cfg;
  float term_lo, term_hi;   // termination threshold bracket (fp32)
  float cap32, om_cap32;    // alpha cap and 1 - cap, rounded
  int fb_test;              // STP_FLAG_FB_TEST: hand every odd item to the float64 pass
  float log_eps;
  int gw, n_items;
  StpOutputs out;
  unsigned long long* counters;
  uint32_t* fb_items;
};

// ---------------------------------------------------------------------------
// float64 resolution paths (rare; kept out of line)

// A comparison level: keys at the Alg. 1 peak of a w x w rect (kind 0), or
// along the ray through a fixed point (kind 1: quad centre, pixel centre).
struct Lvl {
  float x, y;    // rect origin or point (integers / half-integers: exact)
  float w;       // rect size (kind 0)
  int kind;
};
__device__ __forceinline__ Lvl lvl(float x, float y, float w, int kind) {
  Lvl L;
  L.x = x;
  L.y = y;
  L.w = w;
  L.kind = kind;
  return L;
}

// Out-of-line float64 paths take plain pointers (no by-reference kernel
// parameters, which would be copied to the stack).
__device__ __forceinline__ void count_resolve(unsigned long long* counters) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  atomicAdd(counters + C_RES + (smid & 255), 1ull);
}

// key of the reference (tile_culling.py:55-88, 161-195) in float64
__device__ __noinline__ double exact_key(const SplatRec* __restrict__ recs,
                                         const DevCam* __restrict__ cam, uint32_t id, double x,
                                         double y, float w, int kind) {
  const SplatRec& r = recs[id];
  double px = x, py = y;
  if (kind == 0)
    max_point(r.mx, r.my, r.ca, r.cb, r.cc, r.inv_a, r.inv_c, x, y, (double)w, 1.0 / (double)w,
              px, py);
  return key_rec_at(*cam, r, px, py);
}

// (d, rank) order of the reference with float64 keys; empty slots last
__device__ __noinline__ bool exact_less(const SplatRec* __restrict__ recs,
                                        const DevCam* __restrict__ cam,
                                        unsigned long long* counters, double x, double y,
                                        float w, int kind, uint32_t ix, uint32_t iy) {
  if (ix == kNoIdF || iy == kNoIdF) return ix < iy;
  count_resolve(counters);
  const double dx = exact_key(recs, cam, ix, x, y, w, kind);
  const double dy = exact_key(recs, cam, iy, x, y, w, kind);
  return dx < dy || (dx == dy && ix < iy);
}

// eps test of the reference in float64 (hierarchy.py:98-101)
__device__ __noinline__ bool exact_alpha_keep(const SplatRec* __restrict__ recs,
                                              unsigned long long* counters, double eps,
                                              uint32_t id, double px, double py) {
  count_resolve(counters);
  const SplatRec& r = recs[id];
  const double pw = gpower(r.ca, r.cb, r.cc, px - r.mx, py - r.my);
  return (double)r.op * exp_neg(pw, kExp2Tab) >= eps;
}

// certified (x, ix) < (y, iy) in the reference's (key, rank) order
__device__ __forceinline__ bool cless(Key x, uint32_t ix, Key y, uint32_t iy, const FastArgs& A,
                                      const Lvl& L) {
  // |y - x| <= 1 (wrapping is impossible for real keys and kPad)
  if ((uint32_t)(y - x + 1) > 2u) return x < y;
  if (ix == kNoIdF || iy == kNoIdF) return ix < iy;  // empty slots last
  return exact_less(A.recs, A.camp, A.counters, (double)L.x, (double)L.y, L.w, L.kind, ix, iy);
}

// ---------------------------------------------------------------------------
// key at a float64 point (peak / quad centre)
__device__ __forceinline__ Key key_at(const FastArgs& A, uint32_t id, double x, double y) {
  return f2key(__double2float_rn(key_at_point(A.cam, A.r32 + id, x, y)));
}

template <int QH>
struct HeadF {
  Key t[QH];
  float a[QH];
  uint32_t id[QH];
  int n;
};

struct PixelF {
  float px, py;    // pixel centre (exact in fp32)
  double u, w, vn; // camera ray (u, w, 1) and its length
  float T, eT;     // transmittance and its relative error bound
  float C0, C1, C2, D;
  int rc;
  int bad;         // an undecidable termination test was met
  int pix;         // y * W + x, -1 outside the image
};

__device__ __noinline__ void write_record_f(StpOutputs out, int cap, int pix, int rc, float t,
                                            float al, uint32_t id) {
  if (rc < cap && pix >= 0) {
    const int64_t o = (int64_t)pix * cap + rc;
    out.rec_splat[o] = (int32_t)id;
    out.rec_t[o] = t;
    out.rec_alpha[o] = al;
  }
}

// certified termination state: 0 active, 1 terminated, 2 undecidable
__device__ __forceinline__ int tstate(const PixelF& P, const FastArgs& A) {
  const float e = P.eT + 4.0f * kU;
  if (P.T * (1.0f + e) < A.term_lo) return 1;
  if (P.T * (1.0f - e) >= A.term_hi) return 0;
  return 2;
}

// blend (hierarchy.py:81-91)
template <bool REC>
__device__ __forceinline__ void blend_f(PixelF& P, const FastArgs& A, Key tk, float al,
                                        uint32_t id) {
  const int ts = tstate(P, A);
  if (ts != 0) {
    if (ts == 2) P.bad = 1;
    return;
  }
  const float4 oc = __ldg(reinterpret_cast<const float4*>(&A.r32[id].op));
  const float wgt = al * P.T;
  const float t = key2f(tk);
  P.C0 = fmaf(oc.y, wgt, P.C0);
  P.C1 = fmaf(oc.z, wgt, P.C1);
  P.C2 = fmaf(oc.w, wgt, P.C2);
  P.D = fmaf(t, wgt, P.D);
  if (REC) write_record_f(A.out, A.cfg.rec_cap, P.pix, P.rc++, t, al, id);
  P.T = P.T * ((al == A.cap32) ? A.om_cap32 : 1.0f - al);
}

// alpha, eps test, cap and pixel t of one emitted entry (hierarchy.py:94-105):
// the Gaussian exponent and t in float64, alpha fp32 with its error bound.
__device__ __forceinline__ bool emit_eval_f(const PixelF& P, const FastArgs& A, uint32_t id,
                                            Key& t, float& al, float& de) {
  const SplatRec32* r = A.r32 + id;
  const double2 mxy = __ldg(reinterpret_cast<const double2*>(&r->mx));
  const double2 ab = __ldg(reinterpret_cast<const double2*>(&r->ca));
  const double cc = __ldg(&r->cc);
  const float op = __ldg(&r->op);
  const double pw = gpower(ab.x, ab.y, cc, (double)P.px - mxy.x, (double)P.py - mxy.y);
  // alpha >= eps <=> pw <= log(op / eps); thr from MUFU lg2 (|err| < 1e-6 (1 + |thr|))
  const float thr = __logf(op) - A.log_eps;
  const float tolp = fmaf(1e-6f, fabsf(thr), 1e-6f);
  const float pwf = (float)pw;
  if (pwf > thr + tolp) return false;
  if (!(pwf < thr - tolp) &&
      !exact_alpha_keep(A.recs, A.counters, A.cfg.eps, id, (double)P.px, (double)P.py))
    return false;
  al = op * __expf(-pwf);
  // relative error of al vs the reference's float64 alpha: rounding of pw,
  // of pw * log2(e), ex2.approx (2 ulp) and the product
  const float ra = fmaf(2.0f * kU, pwf, 0x1p-21f);
  if (al > A.cap32) al = A.cap32;
  const float om = (al == A.cap32) ? A.om_cap32 : 1.0f - al;
  de = fmaf(fmaf(ra, al, 2.0f * kU), __frcp_ru(om) * 1.0001f, 3.0f * kU);
  t = f2key(__double2float_rn(key_cam(r, P.u, P.w, P.vn)));
  return true;
}

// insort into the pixel queue; on overflow blend the minimum
// (hierarchy.py:110-113); certified comparisons on the pixel ray.
template <int QH, bool EXACT, bool REC>
__device__ __forceinline__ void head_push_f(PixelF& P, HeadF<QH>& H, const FastArgs& A,
                                            const Lvl& L, int qh_rt, Key t, float al, float de,
                                            uint32_t id) {
  // transmittance error of blending this entry, accounted on entry (an upper
  // bound for every termination test that follows)
  P.eT += de;
  const int qh = EXACT ? QH : qh_rt;
  const bool full = H.n >= qh;
  if (full) {
    const bool e_min = cless(t, id, H.t[0], H.id[0], A, L);
    blend_f<REC>(P, A, e_min ? t : H.t[0], e_min ? al : H.a[0], e_min ? id : H.id[0]);
    if (e_min) return;
    int c = 0;
#pragma unroll
    for (int i = 1; i < QH; ++i)
      if ((EXACT || i < qh) && cless(H.t[i], H.id[i], t, id, A, L)) ++c;
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
  // insertion position among the n occupied slots (empty slots follow)
  int c = 0;
#pragma unroll
  for (int i = 0; i < QH; ++i)
    if (i < H.n && cless(H.t[i], H.id[i], t, id, A, L)) ++c;
  H.n++;
#pragma unroll
  for (int i = QH - 1; i >= 0; --i) {
    const int j = i > 0 ? i - 1 : 0;
    const bool take_prev = i > c;
    const bool take_e = i == c;
    H.t[i] = take_prev ? H.t[j] : (take_e ? t : H.t[i]);
    H.a[i] = take_prev ? H.a[j] : (take_e ? al : H.a[i]);
    H.id[i] = take_prev ? H.id[j] : (take_e ? id : H.id[i]);
  }
}

// Bitonic sort of two (key, id) arrays, one element per lane each, ascending;
// array s compares under level Ls.
__device__ __forceinline__ void warp_sort2_f(Key& d0, uint32_t& i0, Key& d1, uint32_t& i1,
                                             int lane, const FastArgs& A, const Lvl& L0,
                                             const Lvl& L1) {
#pragma unroll 1
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      const Key od0 = __shfl_xor_sync(kFull, d0, j);
      const uint32_t oi0 = __shfl_xor_sync(kFull, i0, j);
      const Key od1 = __shfl_xor_sync(kFull, d1, j);
      const uint32_t oi1 = __shfl_xor_sync(kFull, i1, j);
      const bool want_min = (((lane & j) == 0) == ((lane & k) == 0));
      // both lanes of a pair evaluate the same comparison (o < me)
      const bool o_lt0 = cless(od0, oi0, d0, i0, A, L0);
      const bool o_lt1 = cless(od1, oi1, d1, i1, A, L1);
      // take the partner's element when it belongs here
      const bool eq0 = (oi0 == i0), eq1 = (oi1 == i1);
      if (!eq0 && (want_min ? o_lt0 : !o_lt0)) {
        d0 = od0;
        i0 = oi0;
      }
      if (!eq1 && (want_min ? o_lt1 : !o_lt1)) {
        d1 = od1;
        i1 = oi1;
      }
    }
  }
}

// number of (key, id) in sorted a[0..n) strictly below (x, xi)
__device__ __forceinline__ int count_below_f(const Key* ad, const uint32_t* ai, int n, Key x,
                                             uint32_t xi, const FastArgs& A, const Lvl& L) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (cless(ad[m], ai[m], x, xi, A, L)) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// shared-memory queues of one sub-tile (4-byte keys and ids), addressed
// arithmetically:
//   keys [tail0 qt | tail1 qt | batch 32 | mid 4 x qm | scratch 4 x (qm+5) |
//         pad | groups 4 x 17]   ids [same | rings 4 x (R+1)]
// Bank-conflict-free for the 4 quads read by one instruction (mid merge,
// pixel rings): group base 4 banks past the mids, odd strides.
__host__ __device__ inline int fring_size(int qm) { return qm <= 16 ? 64 : 128; }
__host__ __device__ inline int fq_mid0(int qt) { return 2 * qt + 32; }
__host__ __device__ inline int fq_scr0(int qt, int qm) { return fq_mid0(qt) + 4 * qm; }
__host__ __device__ inline int fq_grp0(int qt, int qm) {
  const int b = fq_scr0(qt, qm) + 4 * (qm + 5);
  return b + ((fq_mid0(qt) + 4 - b) & 31);
}
__host__ __device__ inline int fq_ring0(int qt, int qm) { return fq_grp0(qt, qm) + 4 * 17; }
__host__ __device__ inline int fsub_nk(int qt, int qm) { return fq_ring0(qt, qm); }
__host__ __device__ inline size_t fwarp_smem_bytes(int qt, int qm) {
  return (size_t)2 * (2 * fsub_nk(qt, qm) + 4 * (fring_size(qm) + 1)) * 4;
}

struct SubQF {
  Key* d;
  uint32_t* i;
  int qt, qm;
  __device__ __forceinline__ Key* td(int c) const { return d + c * qt; }
  __device__ __forceinline__ uint32_t* ti(int c) const { return i + c * qt; }
  __device__ __forceinline__ Key* bd() const { return d + 2 * qt; }
  __device__ __forceinline__ uint32_t* bi() const { return i + 2 * qt; }
  __device__ __forceinline__ int o_mid(int q) const { return fq_mid0(qt) + q * qm; }
  __device__ __forceinline__ int o_scr(int q) const { return fq_scr0(qt, qm) + q * (qm + 5); }
  __device__ __forceinline__ int o_grp(int q) const { return fq_grp0(qt, qm) + 17 * q; }
  __device__ __forceinline__ uint32_t* ring(int q, int R) const {
    return i + fq_ring0(qt, qm) + q * (R + 1);
  }
};

template <int QH, bool EXACT, int QMX, bool REC>
__global__ void __launch_bounds__(kFThreads, STP_FAST_MINB) k_render_fast(FastArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int qt = A.cfg.q_tail, qm = A.cfg.q_mid, qh_rt = A.cfg.q_head;
  const int R = fring_size(qm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbase = smem_raw + warp * fwarp_smem_bytes(qt, qm);
  const int nk = fsub_nk(qt, qm), ni = fsub_nk(qt, qm) + 4 * (R + 1);
  auto subq = [&](int s) {
    SubQF q;
    q.d = reinterpret_cast<Key*>(wbase) + s * nk;
    q.i = reinterpret_cast<uint32_t*>(wbase) + 2 * nk + s * ni;
    q.qt = qt;
    q.qm = qm;
    return q;
  };
  const int drain_lim = qt - 32;

  const int ps = lane >> 4, pp = lane & 15;
  const int ppx = pp & 3, ppy = pp >> 2;
  const int pq = (ppy >> 1) * 2 + (ppx >> 1);
  const int mq = lane >> 3, mg = (lane >> 1) & 3, mh = lane & 1;

  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  smid &= 255;
  unsigned long long* sm_cnt = A.counters + C_SM + smid;
  unsigned long long* sm_ring = A.counters + C_SMT + smid * 16;

  for (;;) {
    int tile = -1, pair = 0;
    if (lane == 0) {
      const unsigned long long i = atomicAdd(sm_cnt, 1ull);
      const unsigned long long tl = i >> 3;
      pair = (int)(i & 7);
      unsigned long long* slot = sm_ring + (tl & 15);
      if (pair == 0) {
        const int g = (int)atomicAdd(A.counters + C_TILE, 1ull);
        const int gt = g < A.n_items ? g : -1;
        atomicExch(slot, (tl << 32) | (unsigned long long)(gt + 2));
        tile = gt;
      } else {
        unsigned long long v;
        do {
          v = *reinterpret_cast<volatile unsigned long long*>(slot);
        } while ((v >> 32) != tl || (v & 0xffffffffull) == 0);
        tile = (int)(v & 0xffffffffull) - 2;
      }
    }
    tile = __shfl_sync(kFull, tile, 0);
    pair = __shfl_sync(kFull, pair, 0);
    if (tile < 0) break;
    const int tx = tile % A.gw, ty = tile / A.gw;
    const int sx0 = tx * kTile + (pair & 1) * 8, sy0 = ty * kTile + (pair >> 1) * 4;

    PixelF P;
    {
      const int gx = sx0 + ps * 4 + ppx, gy = sy0 + ppy;
      const bool in_img = gx < A.cam.W && gy < A.cam.H;
      P.pix = in_img ? gy * A.cam.W + gx : -1;
      P.px = (float)gx + 0.5f;
      P.py = (float)gy + 0.5f;
      P.u = ((double)P.px - A.cam.cx) * A.cam.inv_fx;
      P.w = ((double)P.py - A.cam.cy) * A.cam.inv_fy;
      const double vv = fma(P.u, P.u, fma(P.w, P.w, 1.0));
      P.vn = vv * frsqrt(vv);
      P.T = in_img ? 1.0f : 0.0f;
      P.eT = 0.0f;
      P.C0 = P.C1 = P.C2 = P.D = 0.f;
      P.rc = 0;
      P.bad = 0;
    }
    HeadF<QH> H;
    H.n = 0;
#pragma unroll
    for (int i = 0; i < QH; ++i) {
      H.t[i] = kPad;
      H.a[i] = 0.f;
      H.id[i] = kNoIdF;
    }

    const uint2 rg = A.ranges[tile];
    const int start = (int)rg.x, k_total = (int)(rg.y - rg.x);
    const double r4y = (double)sy0;

    int cur0 = 0, cur1 = 0, th0 = 0, th1 = 0, nt0 = 0, nt1 = 0, nm0 = 0, nm1 = 0;
    int rh0 = 0, rh1 = 0, rt0 = 0, rt1 = 0;
    bool prod0 = k_total > 0, prod1 = k_total > 0;
    int pos = 0;
    bool abort_item = false;

    // ---- push_mid for sub-tile s (hierarchy.py:147-176)
    auto push_mid = [&](int s) {
      const SubQF Q = subq(s);
      const int cur = s ? cur1 : cur0, th = s ? th1 : th0, nt = s ? nt1 : nt0;
      int nm = s ? nm1 : nm0, rt = s ? rt1 : rt0;
      const int c = min(16, nt);
      const uint32_t* tip = Q.ti(cur) + th;
      const double r2x = (double)(sx0 + 4 * s) + (mq & 1) * 2, r2y = r4y + (mq >> 1) * 2;
      const Lvl L2 = A.cfg.mid_center ? lvl((float)r2x + 1.f, (float)r2y + 1.f, 2.f, 1)
                                      : lvl((float)r2x, (float)r2y, 2.f, 0);
      Key gd[4];
      uint32_t gi[4];
      gd[0] = gd[1] = kPad;
      gi[0] = gi[1] = kNoIdF;
#pragma unroll 1
      for (int u = 0; u < 2; ++u) {
        const int e = 4 * mg + 2 * mh + u;
        if (e < c) {
          const uint32_t sid = tip[e];
          double ptx = (double)L2.x, pty = (double)L2.y;
          if (!A.cfg.mid_center) {
            const SplatRec* r = A.recs + sid;
            const double2 mxy = __ldg(reinterpret_cast<const double2*>(&r->mx));
            const double2 ab = __ldg(reinterpret_cast<const double2*>(&r->ca));
            const double cc = __ldg(&r->cc);
            const double2 inv = __ldg(reinterpret_cast<const double2*>(&r->inv_a));
            max_point(mxy.x, mxy.y, ab.x, ab.y, cc, inv.x, inv.y, r2x, r2y, 2.0, 0.5, ptx, pty);
          }
          const Key dv = key_at(A, sid, ptx, pty);
          if (u) {
            gd[1] = dv;
            gi[1] = sid;
          } else {
            gd[0] = dv;
            gi[0] = sid;
          }
        }
      }
      gd[2] = __shfl_xor_sync(kFull, gd[0], 1);
      gi[2] = __shfl_xor_sync(kFull, gi[0], 1);
      gd[3] = __shfl_xor_sync(kFull, gd[1], 1);
      gi[3] = __shfl_xor_sync(kFull, gi[1], 1);
#define CSWAPF(a, b)                                          \
  if (cless(gd[b], gi[b], gd[a], gi[a], A, L2)) {             \
    const Key td_ = gd[a]; gd[a] = gd[b]; gd[b] = td_;        \
    const uint32_t ti_ = gi[a]; gi[a] = gi[b]; gi[b] = ti_;   \
  }
      CSWAPF(0, 1) CSWAPF(2, 3) CSWAPF(0, 2) CSWAPF(1, 3) CSWAPF(1, 2)
#undef CSWAPF
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
        if (QMX == 8 && qm == 8 && nm == 4 && ng == 4) {
          // steady state (see stp_render.cu): lane slot owns one element
          const bool from_mid = slot0 < 4;
          const int ix = slot0 & 3;
          const Key x = from_mid ? md[ix] : g_d[ix];
          const uint32_t xi = from_mid ? mi[ix] : g_i[ix];
          const Key* od = from_mid ? g_d : md;
          const uint32_t* oi = from_mid ? g_i : mi;
          int rk = ix;
#pragma unroll
          for (int u = 0; u < 4; ++u) rk += cless(od[u], oi[u], x, xi, A, L2);
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
        for (int sl = slot0; sl < L; sl += 8) {
          Key x;
          uint32_t xi;
          int rk;
          if (sl < nm) {
            x = md[sl];
            xi = mi[sl];
            rk = sl;
#pragma unroll 1
            for (int u = 0; u < ng; ++u) rk += cless(g_d[u], g_i[u], x, xi, A, L2);
          } else {
            x = g_d[sl - nm];
            xi = g_i[sl - nm];
            rk = sl - nm;
#pragma unroll 1
            for (int u = 0; u < nm; ++u) rk += cless(md[u], mi[u], x, xi, A, L2);
          }
          sd[rk] = x;
          si[rk] = xi;
        }
        __syncwarp();
        const int h0 = (L >= qm) ? 4 : 0;
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

    const int ring_full = R - 16 - qm;
    for (;;) {
      const int pa = rt0 - rh0, pb = rt1 - rh1;
      const bool ready = (!prod0 || pa >= 16) && (!prod1 || pb >= 16);
      if (pa > ring_full || pb > ring_full || (ready && pa + pb > 0)) {
        // ================= consume
        const int rounds = (pa > 0 && pb > 0) ? min(pa, pb) : max(pa, pb);
        {
          const int pend = ps ? pb : pa;
          const int base = ps ? rh1 : rh0;
          const uint32_t* ring = subq(ps).ring(pq, R);
          for (int e = 0; e < rounds; ++e) {
            const bool live = e < pend && tstate(P, A) == 0;
            FSTAT(4, live);
            if (live) {
              const uint32_t id = ring[(base + e) & (R - 1)];
              Key t;
              float al, de;
              if (emit_eval_f(P, A, id, t, al, de))
                head_push_f<QH, EXACT, REC>(P, H, A, lvl(P.px, P.py, 0.f, 1), qh_rt, t, al,
                                            de, id);
            }
          }
        }
        rh0 += min(rounds, pa);
        rh1 += min(rounds, pb);
        __syncwarp();
        if (__any_sync(kFull, P.bad || (tstate(P, A) == 2))) {
          abort_item = true;
          break;
        }
        continue;
      }
      if (!prod0 && !prod1) break;
      // ================= produce
      const int lim = (pos < k_total) ? drain_lim : 0;
      const bool over0 = prod0 && nt0 > lim, over1 = prod1 && nt1 > lim;
      if (over0 || over1) {
        push_mid((over0 && (!over1 || pa <= pb)) ? 0 : 1);
        continue;
      }
      if (pos < k_total) {
        // termination per sub-tile (hierarchy.py:187-189); all T are decided
        // here (undecidable ones aborted the item after the last consume)
        const unsigned bal = __ballot_sync(kFull, tstate(P, A) == 1);
        if (prod0 && (bal & 0xffffu) == 0xffffu) {
          prod0 = false;
          rh0 = rt0;
        }
        if (prod1 && (bal >> 16) == 0xffffu) {
          prod1 = false;
          rh1 = rt1;
        }
        if (!prod0 && !prod1) continue;
        // ---- load + float64 4x4 cull + fp32 d4 (hierarchy.py:190-199)
        const int j = pos + lane;
        Key dA = kPad, dB = kPad;
        uint32_t iA = kNoIdF, iB = kNoIdF;
        if (j < k_total) {
          const uint32_t sid = A.vals[start + j];
          const SplatRec* r = A.recs + sid;
          const double2 mxy = __ldg(reinterpret_cast<const double2*>(&r->mx));
          const double2 ab = __ldg(reinterpret_cast<const double2*>(&r->ca));
          const double2 ct = make_double2(__ldg(&r->cc), __ldg(&r->thr));
          const double2 inv = __ldg(reinterpret_cast<const double2*>(&r->inv_a));
          const float op = __ldg(&r->op);
#pragma unroll 1
          for (int s = 0; s < 2; ++s) {
            if (s ? !prod1 : !prod0) continue;
            const double r4x = (double)(sx0 + 4 * s);
            double ptx, pty;
            max_point(mxy.x, mxy.y, ab.x, ab.y, ct.x, inv.x, inv.y, r4x, r4y, 4.0, 0.25, ptx,
                      pty);
            if (alpha_keep(gpower(ab.x, ab.y, ct.x, ptx - mxy.x, pty - mxy.y), ct.y, op,
                           A.cfg.eps)) {
              const Key dv = key_at(A, sid, ptx, pty);
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
        pos += 32;
        const int nkA = __popc(__ballot_sync(kFull, iA != kNoIdF));
        const int nkB = __popc(__ballot_sync(kFull, iB != kNoIdF));
        if (nkA + nkB == 0) continue;
        warp_sort2_f(dA, iA, dB, iB, lane, A, lvl((float)sx0, (float)sy0, 4.f, 0),
                     lvl((float)(sx0 + 4), (float)sy0, 4.f, 0));
        // ---- merge each sorted batch into its tail (heap_merge, :201)
#pragma unroll 1
        for (int s = 0; s < 2; ++s) {
          const int nks = s ? nkB : nkA;
          if (nks == 0) continue;
          const Key ds = s ? dB : dA;
          const uint32_t is = s ? iB : iA;
          const SubQF Q = subq(s);
          const int cur = s ? cur1 : cur0, th = s ? th1 : th0, nt = s ? nt1 : nt0;
          Q.bd()[lane] = ds;
          Q.bi()[lane] = is;
          __syncwarp();
          const Key* td = Q.td(cur) + th;
          const uint32_t* ti = Q.ti(cur) + th;
          Key* od = Q.td(cur ^ 1);
          uint32_t* oi = Q.ti(cur ^ 1);
          if (lane < nks) {
            const int rk =
                count_below_f(td, ti, nt, ds, is, A, lvl((float)(sx0 + 4 * s), (float)sy0, 4.f, 0));
            od[lane + rk] = ds;
            oi[lane + rk] = is;
          }
          for (int t = lane; t < nt; t += 32) {
            const int rk = count_below_f(Q.bd(), Q.bi(), nks, td[t], ti[t], A,
                                         lvl((float)(sx0 + 4 * s), (float)sy0, 4.f, 0));
            od[t + rk] = td[t];
            oi[t + rk] = ti[t];
          }
          __syncwarp();
          if (s) {
            cur1 ^= 1;
            th1 = 0;
            nt1 += nks;
          } else {
            cur0 ^= 1;
            th0 = 0;
            nt0 += nks;
          }
        }
        continue;
      }
      // ---- end of the bin, tails empty: flush a sub-tile's mid queues
      {
        const int fs = prod0 ? 0 : 1;
        const SubQF Q = subq(fs);
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
    if (!abort_item) {
      // heads drain in ascending (t, rank) (hierarchy.py:215-217)
#pragma unroll
      for (int i = 0; i < QH; ++i)
        if (i < H.n) blend_f<REC>(P, A, H.t[i], H.a[i], H.id[i]);
      abort_item = __any_sync(kFull, P.bad);
    }
    if (A.fb_test && ((tile + pair) & 1)) abort_item = true;
    if (abort_item) {
      // undecidable termination: the float64 kernel renders this pair
      if (lane == 0) {
        const unsigned long long k = atomicAdd(A.counters + C_FB, 1ull);
        A.fb_items[k] = (uint32_t)(tile * 8 + pair);
      }
      continue;
    }
    if (P.pix >= 0) {
      const float T = P.T;
      const float c0 = P.C0 + (float)((double)P.T * A.cfg.bg[0]);
      const float c1 = P.C1 + (float)((double)P.T * A.cfg.bg[1]);
      const float c2 = P.C2 + (float)((double)P.T * A.cfg.bg[2]);
      A.out.color[(int64_t)P.pix * 3 + 0] = c0;
      A.out.color[(int64_t)P.pix * 3 + 1] = c1;
      A.out.color[(int64_t)P.pix * 3 + 2] = c2;
      A.out.transmittance[P.pix] = T;
      if (A.out.depth) A.out.depth[P.pix] = P.D;
      if (REC) A.out.rec_count[P.pix] = P.rc;
      if (!(isfinite(c0) && isfinite(c1) && isfinite(c2) && isfinite(T)))
        atomicAdd(A.counters + C_NONFINITE, 1ull);
    }
  }
}

size_t render_fast_smem_bytes(int qt, int qm) {
  return kFWarpsPerBlock * fwarp_smem_bytes(qt, qm);
}

template <int QH, bool EXACT, int QMX, bool REC>
static void launch_fast_t(const FastArgs& A, size_t smem, cudaStream_t s) {
  static size_t attr = 0;
  static int blocks_per_sm = 0, n_sm = 0;
  if (smem != attr || blocks_per_sm == 0) {
    cudaFuncSetAttribute(k_render_fast<QH, EXACT, QMX, REC>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_render_fast<QH, EXACT, QMX, REC>,
                                                  kFThreads, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int want = (A.n_items * 8 + kFWarpsPerBlock - 1) / kFWarpsPerBlock;
  const int grid = min(want, n_sm * blocks_per_sm);
  if (grid > 0) k_render_fast<QH, EXACT, QMX, REC><<<grid, kFThreads, smem, s>>>(A);
}

void launch_render_fast(const Frame& f, int buf, const StpOutputs& out, cudaStream_t s) {
  FastArgs A;
  A.recs = f.recs;
  A.r32 = f.recs32;
  A.vals = f.vals;
  A.ranges = f.ranges;
  A.camp = f.camp;
  A.cam = f.cam;
  A.cfg = f.cfg;
  A.term_lo = (float)(f.cfg.term * (1.0 - 0x1p-22));
  A.term_hi = (float)(f.cfg.term * (1.0 + 0x1p-22));
  A.cap32 = (float)f.cfg.cap;
  A.om_cap32 = (float)(1.0 - f.cfg.cap);
  A.fb_test = f.fb_test;
  A.log_eps = (float)log(f.cfg.eps);
  A.gw = f.gw;
  A.n_items = f.n_tiles;
  A.out = out;
  A.counters = f.counters;
  A.fb_items = f.fb_items;
  const size_t smem = render_fast_smem_bytes(f.cfg.q_tail, f.cfg.q_mid);
  if (f.cfg.rec_cap > 0) {  // debug records: generic instantiation
    if (f.cfg.q_mid > 8) launch_fast_t<16, false, 0, true>(A, smem, s);
    else launch_fast_t<16, false, 8, true>(A, smem, s);
    return;
  }
  if (f.cfg.q_mid > 8) {
    launch_fast_t<16, false, 0, false>(A, smem, s);
    return;
  }
  switch (f.cfg.q_head) {
    case 1: launch_fast_t<1, true, 8, false>(A, smem, s); break;
    case 2: launch_fast_t<2, true, 8, false>(A, smem, s); break;
    case 4: launch_fast_t<4, true, 8, false>(A, smem, s); break;
    case 8: launch_fast_t<8, true, 8, false>(A, smem, s); break;
    case 16: launch_fast_t<16, true, 8, false>(A, smem, s); break;
    default: launch_fast_t<16, false, 8, false>(A, smem, s); break;
  }
}

}  // namespace stp
