// K6: hierarchical resort + front-to-back blend, one CTA per 16x16 tile.
//
// Exact restatement of hierarchy.render_tile (hierarchy.py:27-219; contract in
// SURVEY.md Appendix A).  One warp owns two horizontally adjacent 4x4
// sub-tiles; half-warp s = lane>>4 is sub-tile s, lane&15 its pixel.
//
//   load   : lane l evaluates bin entry pos+l against both 4x4 rects
//            (max_points + alpha test + t_opt on the peak ray, float64),
//            hierarchy.py:190-199
//   sort   : warp bitonic network on (d4, rank) for both sub-tiles at once,
//            merged into the tail queue kept in shared memory (:200-207)
//   drain  : while len(tail) > q_tail - 32 pop 16 -> push_mid (:178-182)
//   mid    : lane (s, quad, group) re-keys 4 entries at its 2x2 rect, sorts
//            them, and the four groups of a quad merge into its mid queue in
//            order, popping 4 at a time while len(mid) >= q_mid (:147-176)
//   pixel  : every lane consumes its quad's emitted stream: alpha, eps test,
//            cap, pixel-ray t_opt, register insertion queue of q_head,
//            blending the minimum on overflow (:93-113, 81-91)
//   drain  : tail -> mids -> heads at the end of the bin (:210-217)
//
// Termination (:187-189) is checked per batch for the warp's 32 pixels; a
// terminated pixel's blends are no-ops, so stopping at warp granularity is
// output-identical.  Sub-tiles / quads outside the image run the same queues
// (their rects stay full size, hierarchy.py:124-142) and write nothing.
#include "stp_common.cuh"

namespace stp {

constexpr int kRenderThreads = 256;  // 8 warps = 16 sub-tiles = one tile
constexpr unsigned kNoId = 0xffffffffu;

__device__ __forceinline__ bool lt(double da, uint32_t ia, double db, uint32_t ib) {
  return da < db || (da == db && ia < ib);
}

// Per-warp shared-memory queues for the two sub-tiles, addressed
// arithmetically (no runtime-indexed pointer arrays): per sub-tile s a double
// block [tail0 qt | tail1 qt | batch 32 | mid 4*qm | scratch 4*(qm+4)] and an
// id block [tail0 | tail1 | batch | mid | scratch | emitted 4*emcap], then
// the small counters nm[2][4], ne[2][4].
struct WarpQ {
  double* dbase;
  uint32_t* ibase;
  int* cnt;
  int qt, qm, emcap, ds, is;
  __device__ __forceinline__ double* td(int s, int c) const { return dbase + s * ds + c * qt; }
  __device__ __forceinline__ uint32_t* ti(int s, int c) const { return ibase + s * is + c * qt; }
  __device__ __forceinline__ double* bd(int s) const { return dbase + s * ds + 2 * qt; }
  __device__ __forceinline__ uint32_t* bi(int s) const { return ibase + s * is + 2 * qt; }
  __device__ __forceinline__ double* md(int s, int q) const { return dbase + s * ds + 2 * qt + 32 + q * qm; }
  __device__ __forceinline__ uint32_t* mi(int s, int q) const { return ibase + s * is + 2 * qt + 32 + q * qm; }
  __device__ __forceinline__ double* sd(int s, int q) const {
    return dbase + s * ds + 2 * qt + 32 + 4 * qm + q * (qm + 4);
  }
  __device__ __forceinline__ uint32_t* si(int s, int q) const {
    return ibase + s * is + 2 * qt + 32 + 4 * qm + q * (qm + 4);
  }
  __device__ __forceinline__ uint32_t* em(int s, int q) const {
    return ibase + s * is + 2 * qt + 32 + 4 * qm + 4 * (qm + 4) + q * emcap;
  }
  __device__ __forceinline__ int& nm(int s, int q) const { return cnt[s * 4 + q]; }
  __device__ __forceinline__ int& ne(int s, int q) const { return cnt[8 + s * 4 + q]; }
};

__host__ __device__ inline int emit_cap(int qm) { return qm + 20; }
__host__ __device__ inline int q_ds(int qt, int qm) { return 2 * qt + 32 + 4 * qm + 4 * (qm + 4); }
__host__ __device__ inline int q_is(int qt, int qm) { return q_ds(qt, qm) + 4 * emit_cap(qm); }

__host__ __device__ inline size_t warp_smem_bytes(int qt, int qm) {
  size_t b = 2 * (size_t)q_ds(qt, qm) * 8 + 2 * (size_t)q_is(qt, qm) * 4 + 16 * 4;
  return (b + 15) & ~(size_t)15;
}

__device__ inline WarpQ carve(unsigned char* base, int qt, int qm) {
  WarpQ q;
  q.qt = qt;
  q.qm = qm;
  q.emcap = emit_cap(qm);
  q.ds = q_ds(qt, qm);
  q.is = q_is(qt, qm);
  q.dbase = reinterpret_cast<double*>(base);
  q.ibase = reinterpret_cast<uint32_t*>(q.dbase + 2 * q.ds);
  q.cnt = reinterpret_cast<int*>(q.ibase + 2 * q.is);
  return q;
}

template <int QH>
struct Head {
  double t[QH];
  double a[QH];
  uint32_t id[QH];
  float c0[QH], c1[QH], c2[QH];
  int n;
};

struct Pixel {
  double px, py;
  double d0, d1, d2;            // unit pixel ray (rasterizer.py:405)
  double f[6];                  // ray features (rasterizer.py:406)
  double T;                     // transmittance (float64: the termination test)
  float C0, C1, C2, D;
  int rc;                       // records written
  bool in_img;
  int64_t pix;                  // y * W + x
};

struct RenderArgs {
  const SplatRec* __restrict__ recs;
  const uint32_t* __restrict__ vals;
  const uint2* __restrict__ ranges;
  DevCam cam;
  DevCfg cfg;
  int gw;
  StpOutputs out;
  unsigned long long* counters;
};

__device__ __forceinline__ void blend(Pixel& P, const RenderArgs& A, double t, double al,
                                      uint32_t id, float c0, float c1, float c2) {
  // hierarchy.py:81-91
  if (P.T < A.cfg.term) return;
  const double w = al * P.T;
  const float wf = (float)w;
  P.C0 += c0 * wf;
  P.C1 += c1 * wf;
  P.C2 += c2 * wf;
  P.D += (float)(t * w);
  if (A.cfg.rec_cap > 0 && P.in_img) {
    if (P.rc < A.cfg.rec_cap) {
      const int64_t o = P.pix * A.cfg.rec_cap + P.rc;
      A.out.rec_splat[o] = (int32_t)id;
      A.out.rec_t[o] = (float)t;
      A.out.rec_alpha[o] = (float)al;
    }
    P.rc++;
  }
  P.T = P.T * (1.0 - al);
}

// emit_to_pixel (hierarchy.py:93-113) for one entry.
template <int QH>
__device__ __forceinline__ void emit(Pixel& P, Head<QH>& H, const RenderArgs& A, int qh,
                                     uint32_t id) {
  const SplatRec* r = A.recs + id;
  const double2 mxy = __ldg(reinterpret_cast<const double2*>(&r->mx));
  const double2 ab = __ldg(reinterpret_cast<const double2*>(&r->ca));
  const double2 ct = __ldg(reinterpret_cast<const double2*>(&r->cc));
  const double dx = P.px - mxy.x, dy = P.py - mxy.y;
  const double pw = gpower(ab.x, ab.y, ct.x, dx, dy);
  if (pw > ct.y + 1e-9) return;  // alpha < eps far from the boundary
  const float4 oc = __ldg(reinterpret_cast<const float4*>(&r->op));
  double al = (double)oc.x * exp(-pw);
  if (al < A.cfg.eps) return;
  if (al > A.cfg.cap) al = A.cfg.cap;
  const double2 m01 = __ldg(reinterpret_cast<const double2*>(&r->m[0]));
  const double2 m23 = __ldg(reinterpret_cast<const double2*>(&r->m[2]));
  const double2 m45 = __ldg(reinterpret_cast<const double2*>(&r->m[4]));
  const double2 q01 = __ldg(reinterpret_cast<const double2*>(&r->q0));
  const double q2 = __ldg(&r->q2);
  const double num = P.d0 * q01.x + P.d1 * q01.y + P.d2 * q2;
  const double den = P.f[0] * m01.x + P.f[1] * m01.y + P.f[2] * m23.x + P.f[3] * m23.y +
                     P.f[4] * m45.x + P.f[5] * m45.y;
  const double t = num / den;
  // insort + pop-min-on-overflow
  if (H.n < qh) {
    bool placed = false;
#pragma unroll
    for (int i = QH - 1; i >= 0; --i) {
      if (i > H.n) continue;
      if (i > 0 && lt(t, id, H.t[i - 1], H.id[i - 1])) {
        H.t[i] = H.t[i - 1];
        H.a[i] = H.a[i - 1];
        H.id[i] = H.id[i - 1];
        H.c0[i] = H.c0[i - 1];
        H.c1[i] = H.c1[i - 1];
        H.c2[i] = H.c2[i - 1];
      } else if (!placed) {
        H.t[i] = t;
        H.a[i] = al;
        H.id[i] = id;
        H.c0[i] = oc.y;
        H.c1[i] = oc.z;
        H.c2[i] = oc.w;
        placed = true;
      }
    }
    H.n++;
  } else if (lt(t, id, H.t[0], H.id[0])) {
    blend(P, A, t, al, id, oc.y, oc.z, oc.w);
  } else {
    blend(P, A, H.t[0], H.a[0], H.id[0], H.c0[0], H.c1[0], H.c2[0]);
    bool placed = false;
#pragma unroll
    for (int i = 0; i < QH; ++i) {
      if (i >= qh || placed) continue;
      const bool last = (i + 1 >= qh) || (i + 1 >= QH);
      if (last || lt(t, id, H.t[(i + 1 < QH) ? i + 1 : i], H.id[(i + 1 < QH) ? i + 1 : i])) {
        H.t[i] = t;
        H.a[i] = al;
        H.id[i] = id;
        H.c0[i] = oc.y;
        H.c1[i] = oc.z;
        H.c2[i] = oc.w;
        placed = true;
      } else {
        const int j = (i + 1 < QH) ? i + 1 : i;
        H.t[i] = H.t[j];
        H.a[i] = H.a[j];
        H.id[i] = H.id[j];
        H.c0[i] = H.c0[j];
        H.c1[i] = H.c1[j];
        H.c2[i] = H.c2[j];
      }
    }
  }
}

// Bitonic sort of one (d, id) pair per lane, ascending across the warp.
__device__ __forceinline__ void warp_sort2(double& d0, uint32_t& i0, double& d1, uint32_t& i1,
                                           int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const double od0 = shfl_xor_d(d0, j);
      const uint32_t oi0 = __shfl_xor_sync(kFull, i0, j);
      const double od1 = shfl_xor_d(d1, j);
      const uint32_t oi1 = __shfl_xor_sync(kFull, i1, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      const bool want_min = (lower == up);
      const bool o_less0 = lt(od0, oi0, d0, i0);
      const bool o_less1 = lt(od1, oi1, d1, i1);
      if (want_min ? o_less0 : (!o_less0 && !(od0 == d0 && oi0 == i0))) {
        d0 = od0;
        i0 = oi0;
      }
      if (want_min ? o_less1 : (!o_less1 && !(od1 == d1 && oi1 == i1))) {
        d1 = od1;
        i1 = oi1;
      }
    }
  }
}

// number of (d,id) in sorted array a[0..n) strictly below (x, xi)
__device__ __forceinline__ int count_below(const double* ad, const uint32_t* ai, int n, double x,
                                           uint32_t xi) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (lt(ad[m], ai[m], x, xi)) lo = m + 1;
    else hi = m;
  }
  return lo;
}

template <int QH>
__global__ void __launch_bounds__(kRenderThreads) k_render(RenderArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int qt = A.cfg.q_tail, qm = A.cfg.q_mid, qh = A.cfg.q_head;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const WarpQ Q = carve(smem_raw + warp * warp_smem_bytes(qt, qm), qt, qm);

  const int tile = blockIdx.x;
  const int tx = tile % A.gw, ty = tile / A.gw;
  const int x0 = tx * kTile, y0 = ty * kTile;
  const int sr = warp >> 1, sc = (warp & 1) * 2;  // sub-tile row, first sub-tile column
  const double term = A.cfg.term;

  // this lane's pixel
  Pixel P;
  const int ps = lane >> 4, pp = lane & 15, ppx = pp & 3, ppy = pp >> 2;
  const int pq = (ppy >> 1) * 2 + (ppx >> 1);
  {
    const int gx = x0 + (sc + ps) * 4 + ppx, gy = y0 + sr * 4 + ppy;
    P.in_img = gx < A.cam.W && gy < A.cam.H;
    P.pix = (int64_t)gy * A.cam.W + gx;
    P.px = (double)gx + 0.5;
    P.py = (double)gy + 0.5;
    ray_dir(A.cam, P.px, P.py, P.d0, P.d1, P.d2);
    P.f[0] = P.d0 * P.d0;
    P.f[1] = P.d1 * P.d1;
    P.f[2] = P.d2 * P.d2;
    P.f[3] = 2 * P.d0 * P.d1;
    P.f[4] = 2 * P.d0 * P.d2;
    P.f[5] = 2 * P.d1 * P.d2;
    P.T = P.in_img ? 1.0 : 0.0;
    P.C0 = P.C1 = P.C2 = P.D = 0.f;
    P.rc = 0;
  }
  Head<QH> H;
  H.n = 0;

  const uint2 rg = A.ranges[tile];
  const int start = (int)rg.x, k_total = (int)(rg.y - rg.x);

  if (k_total > 0) {
    // 4x4 rects of the two sub-tiles (hierarchy.py:124-127), always full size
    double r4x[2], r4y[2];
    r4x[0] = (double)(x0 + sc * 4);
    r4x[1] = (double)(x0 + (sc + 1) * 4);
    const double r4y0 = (double)(y0 + sr * 4);
    r4y[0] = r4y[1] = r4y0;
    // push_mid lane role: (sub s, quad q, group g)
    const int ms = lane >> 4, mq = (lane >> 2) & 3, mg = lane & 3;
    const double r2x0 = r4x[ms] + (mq & 1) * 2, r2y0 = r4y0 + (mq >> 1) * 2;

    // tail state per sub-tile (warp-uniform): ping-pong buffer, head, length
    int cur0 = 0, cur1 = 0, th0 = 0, th1 = 0, nt0 = 0, nt1 = 0;
    if (lane < 16) Q.cnt[lane] = 0;
    __syncwarp();

    // push_mid for chunk sizes c[0], c[1] taken from the tail fronts
    auto push_mid = [&](int c0, int c1) {
      const int ce = ms ? c1 : c0;
      double gd[4];
      uint32_t gi[4];
      const uint32_t* tip = Q.ti(ms, ms ? cur1 : cur0) + (ms ? th1 : th0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = 4 * mg + u;
        gd[u] = INFINITY;
        gi[u] = kNoId;
        if (e < ce) {
          const uint32_t id = tip[e];
          const SplatRec* r = A.recs + id;
          double ptx, pty;
          if (A.cfg.mid_center) {
            ptx = r2x0 + 1.0;
            pty = r2y0 + 1.0;
          } else {
            max_point(r->mx, r->my, r->ca, r->cb, r->cc, r2x0, r2x0 + 2.0, r2y0, r2y0 + 2.0, ptx,
                      pty);
          }
          double d0, d1, d2;
          ray_dir(A.cam, ptx, pty, d0, d1, d2);
          gd[u] = blend_depth(r->m, r->q0, r->q1, r->q2, d0, d1, d2);
          gi[u] = id;
        }
      }
      // sort the group of 4 (sorting network)
#define CSWAP(a, b)                                  \
  if (lt(gd[b], gi[b], gd[a], gi[a])) {              \
    const double td_ = gd[a]; gd[a] = gd[b]; gd[b] = td_; \
    const uint32_t ti_ = gi[a]; gi[a] = gi[b]; gi[b] = ti_; \
  }
      CSWAP(0, 1) CSWAP(2, 3) CSWAP(0, 2) CSWAP(1, 3) CSWAP(1, 2)
#undef CSWAP
      // groups merge into the quad's mid queue in order
      for (int gg = 0; gg < 4; ++gg) {
        if (mg == gg && 4 * gg < ce) {
          const int ng = min(4, ce - 4 * gg);
          double* md = Q.md(ms, mq);
          uint32_t* mi = Q.mi(ms, mq);
          double* sd = Q.sd(ms, mq);
          uint32_t* si = Q.si(ms, mq);
          uint32_t* em = Q.em(ms, mq);
          const int n = Q.nm(ms, mq);
          int ne = Q.ne(ms, mq);
          // two-pointer merge mid[0..n) with group[0..ng)
          int a = 0, o = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if (b >= ng) break;
            while (a < n && lt(md[a], mi[a], gd[b], gi[b])) {
              sd[o] = md[a];
              si[o] = mi[a];
              ++o;
              ++a;
            }
            sd[o] = gd[b];
            si[o] = gi[b];
            ++o;
          }
          while (a < n) {
            sd[o] = md[a];
            si[o] = mi[a];
            ++o;
            ++a;
          }
          // while len(mid) >= q_mid: flush_mid pops 4 (hierarchy.py:168-176)
          int h0 = 0;
          while (o - h0 >= qm) {
            for (int u = 0; u < 4; ++u) em[ne++] = si[h0 + u];
            h0 += 4;
          }
          for (int u = h0; u < o; ++u) {
            md[u - h0] = sd[u];
            mi[u - h0] = si[u];
          }
          Q.nm(ms, mq) = o - h0;
          Q.ne(ms, mq) = ne;
        }
        __syncwarp();
      }
    };

    // consume the emitted streams
    auto pixel_phase = [&]() {
      __syncwarp();
      const int n = Q.ne(ps, pq);
      int nmax = n;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nmax = max(nmax, __shfl_xor_sync(kFull, nmax, o));
      const uint32_t* em = Q.em(ps, pq);
      for (int e = 0; e < nmax; ++e)
        if (e < n) emit<QH>(P, H, A, qh, em[e]);
      __syncwarp();
      if (lane < 8) Q.cnt[8 + lane] = 0;
      __syncwarp();
    };

    const int drain_lim = qt - 32;  // drain_tail(q_tail - batch_load)
    bool stopped = false;
    for (int pos = 0; pos < k_total; pos += 32) {
      if (__all_sync(kFull, P.T < term)) {
        stopped = true;
        break;
      }
      // ---- load + 4x4 cull + d4 (hierarchy.py:190-199)
      const int j = pos + lane;
      double d[2] = {INFINITY, INFINITY};
      uint32_t ids[2] = {kNoId, kNoId};
      if (j < k_total) {
        const uint32_t id = A.vals[start + j];
        const SplatRec* r = A.recs + id;
        const double2 mxy = __ldg(reinterpret_cast<const double2*>(&r->mx));
        const double2 ab = __ldg(reinterpret_cast<const double2*>(&r->ca));
        const double2 ct = __ldg(reinterpret_cast<const double2*>(&r->cc));
        const float op = __ldg(&r->op);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          double ptx, pty;
          max_point(mxy.x, mxy.y, ab.x, ab.y, ct.x, r4x[s], r4x[s] + 4.0, r4y[s], r4y[s] + 4.0,
                    ptx, pty);
          if (alpha_keep(gpower(ab.x, ab.y, ct.x, ptx - mxy.x, pty - mxy.y), ct.y, op,
                         A.cfg.eps)) {
            double d0, d1, d2;
            ray_dir(A.cam, ptx, pty, d0, d1, d2);
            d[s] = blend_depth(r->m, r->q0, r->q1, r->q2, d0, d1, d2);
            ids[s] = id;
          }
        }
      }
      warp_sort2(d[0], ids[0], d[1], ids[1], lane);
      int nk[2];
      nk[0] = __popc(__ballot_sync(kFull, ids[0] != kNoId));
      nk[1] = __popc(__ballot_sync(kFull, ids[1] != kNoId));
      Q.bd(0)[lane] = d[0];
      Q.bi(0)[lane] = ids[0];
      Q.bd(1)[lane] = d[1];
      Q.bi(1)[lane] = ids[1];
      __syncwarp();
      // ---- merge the sorted batch into the tail (heap_merge, :201)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int nks = nk[s];
        if (nks == 0) continue;
        const int cs = s ? cur1 : cur0, ths = s ? th1 : th0, nts = s ? nt1 : nt0;
        const double* td = Q.td(s, cs) + ths;
        const uint32_t* ti = Q.ti(s, cs) + ths;
        double* od = Q.td(s, cs ^ 1);
        uint32_t* oi = Q.ti(s, cs ^ 1);
        if (lane < nks) {
          const int r = count_below(td, ti, nts, d[s], ids[s]);
          od[lane + r] = d[s];
          oi[lane + r] = ids[s];
        }
        for (int t = lane; t < nts; t += 32) {
          const int r = count_below(Q.bd(s), Q.bi(s), nks, td[t], ti[t]);
          od[t + r] = td[t];
          oi[t + r] = ti[t];
        }
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
      __syncwarp();
      // ---- drain_tail(q_tail - 32): pop 16 while len > limit
      while (nt0 > drain_lim || nt1 > drain_lim) {
        const int c0 = nt0 > drain_lim ? 16 : 0;
        const int c1 = nt1 > drain_lim ? 16 : 0;
        push_mid(c0, c1);
        th0 += c0;
        nt0 -= c0;
        th1 += c1;
        nt1 -= c1;
        pixel_phase();
      }
    }
    if (!stopped) {
      // ---- end of stream (hierarchy.py:210-217)
      while (nt0 > 0 || nt1 > 0) {
        const int c0 = min(16, nt0), c1 = min(16, nt1);
        push_mid(c0, c1);
        th0 += c0;
        nt0 -= c0;
        th1 += c1;
        nt1 -= c1;
        pixel_phase();
      }
      // flush every mid queue completely, in order
      if (mg == 0) {
        const int n = Q.nm(ms, mq);
        uint32_t* em = Q.em(ms, mq);
        const uint32_t* mi = Q.mi(ms, mq);
        int ne = Q.ne(ms, mq);
        for (int u = 0; u < n; ++u) em[ne++] = mi[u];
        Q.ne(ms, mq) = ne;
        Q.nm(ms, mq) = 0;
      }
      pixel_phase();
      // heads drain in ascending (t, rank)
#pragma unroll
      for (int i = 0; i < QH; ++i)
        if (i < H.n) blend(P, A, H.t[i], H.a[i], H.id[i], H.c0[i], H.c1[i], H.c2[i]);
    }
  }

  if (P.in_img) {
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

template <int QH>
static void launch_render_t(const RenderArgs& A, int n_tiles, size_t smem, cudaStream_t s) {
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(k_render<QH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  k_render<QH><<<n_tiles, kRenderThreads, smem, s>>>(A);
}

size_t render_smem_bytes(int qt, int qm) { return 8 * warp_smem_bytes(qt, qm); }

void launch_render(const Frame& f, int buf, const StpOutputs& out, cudaStream_t s) {
  RenderArgs A;
  A.recs = f.recs;
  A.vals = f.vals[buf];
  A.ranges = f.ranges;
  A.cam = f.cam;
  A.cfg = f.cfg;
  A.gw = f.gw;
  A.out = out;
  A.counters = f.counters;
  const size_t smem = render_smem_bytes(f.cfg.q_tail, f.cfg.q_mid);
  if (f.cfg.q_head <= 4) launch_render_t<4>(A, f.n_tiles, smem, s);
  else if (f.cfg.q_head <= 8) launch_render_t<8>(A, f.n_tiles, smem, s);
  else launch_render_t<16>(A, f.n_tiles, smem, s);
}

}  // namespace stp
