// K0 frame init, K1 preprocess, K2 scan, K3 duplicate.
//
// K1 restates project_scene (gaussian_math.py:323-434) per Gaussian in
// float64 from the float32 inputs, plus the coarse tile rect
// (rasterizer.py:307-321) and the exact-culled tile count
// (rasterizer.py:334-339).  K3 re-enumerates the surviving tiles and writes
// (key = tile<<32 | fp32-orderable t_opt at the 16x16 peak, value = Gaussian
// id) in Gaussian order (rasterizer.py:328-350), so a stable LSD sort breaks
// key ties by rank exactly like np.lexsort((rank, key, tile)).
//
// The (splat, tile) pairs of a warp's 32 splats are enumerated cooperatively
// (warp_expand), so lanes stay busy whatever the rect sizes (the paper's
// load balancing, applied to every splat).
#include <atomic>

#include "stp_common.cuh"

namespace stp {

#ifndef STP_PRE_THREADS
#define STP_PRE_THREADS 64  // 64-thread K1/K3 blocks, 16 per SM: K1 0.284 -> 0.270 ms (profiles/r3h; 128: 0.275, 512: 0.309)
#endif
constexpr int kPreThreads = STP_PRE_THREADS;
constexpr int kMaskTiles = 64;  // rects up to this many tiles carry a survivor mask (K1 -> K3)
// masks[] value of a Gaussian K1 listed for the row kernels (rect > 64 tiles)
constexpr unsigned long long kRowsListed = ~0ull;
#ifndef STP_K1_MINB
#define STP_K1_MINB (1024 / STP_PRE_THREADS)  // 64 registers, 32 warps per SM (measured K1 0.35 -> 0.33 ms at 256 x 4)
#endif
#ifndef STP_SPLIT_SH
#define STP_SPLIT_SH 0
#endif
#ifndef STP_K1_V2
#define STP_K1_V2 1  // register-lean projection + streaming record stores
#endif
#ifndef STP_K1_HOIST
#define STP_K1_HOIST 1  // all input loads issued before the cull tests
#endif
#ifndef STP_K1_SH_EARLY
#define STP_K1_SH_EARLY 0  // SH colour before the covariance algebra (needs HOIST)
#endif

__constant__ double c_SH_C0 = 0.28209479177387814;
__constant__ double c_SH_C1 = 0.4886025119029199;
__constant__ double c_SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                  -1.0925484305920792, 0.5462742152960396};
__constant__ double c_SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                  0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                                  -0.5900435899266435};

// ---------------------------------------------------------------------------
// K0: zero the per-frame counters / histograms / tile ranges, bump the epoch
// that tags the sort's look-back words (so they never need clearing).
__global__ void k_init(unsigned long long* counters, uint32_t* hist, int hist_n, uint2* ranges,
                       int n_tiles, DevCam cam, DevCam* camp, unsigned long long epoch) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = gridDim.x * blockDim.x;
  if (tid == 0) {
    // process-wide frame number: look-back words left in a recycled
    // workspace buffer (another workspace's frames) can never match it
    counters[C_EPOCH] = epoch;
    *camp = cam;
  }
  for (int i = tid; i < C_COUNT; i += stride)
    if (i != C_EPOCH) counters[i] = 0;
  for (int i = tid; i < hist_n; i += stride) hist[i] = 0;
  for (int i = tid; i < n_tiles; i += stride) ranges[i] = make_uint2(0, 0);
}

// ---------------------------------------------------------------------------
// K1 preprocess.

// SH colour (gaussian_math.py:152-175, 415-419) in fp32: the colour feeds
// only the blended pixel values (no decision), where fp32 rounding (~1e-7)
// is far inside the 1e-4 output tolerance.
__device__ __forceinline__ void sh_color(const float* __restrict__ sh, int K, float x, float y,
                                         float z, float out[3]) {
  float b[16];
  const float xx = x * x, yy = y * y, zz = z * z;
  const float xy = x * y, yz = y * z, xz = x * z;
  b[0] = (float)c_SH_C0;
  if (K > 1) {
    b[1] = -(float)c_SH_C1 * y;
    b[2] = (float)c_SH_C1 * z;
    b[3] = -(float)c_SH_C1 * x;
  }
  if (K > 4) {
    b[4] = (float)c_SH_C2[0] * xy;
    b[5] = (float)c_SH_C2[1] * yz;
    b[6] = (float)c_SH_C2[2] * (2.0f * zz - xx - yy);
    b[7] = (float)c_SH_C2[3] * xz;
    b[8] = (float)c_SH_C2[4] * (xx - yy);
  }
  if (K > 9) {
    b[9] = (float)c_SH_C3[0] * y * (3.0f * xx - yy);
    b[10] = (float)c_SH_C3[1] * xy * z;
    b[11] = (float)c_SH_C3[2] * y * (4.0f * zz - xx - yy);
    b[12] = (float)c_SH_C3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = (float)c_SH_C3[4] * x * (4.0f * zz - xx - yy);
    b[14] = (float)c_SH_C3[5] * z * (xx - yy);
    b[15] = (float)c_SH_C3[6] * x * (xx - 3.0f * yy);
  }
  float acc[3] = {0.5f, 0.5f, 0.5f};
  if (K == 16) {
    // 192 B per Gaussian: 12 x float4, consumed as they arrive
    const float4* p = reinterpret_cast<const float4*>(sh);
#pragma unroll
    for (int u = 0; u < 12; ++u) {
      const float4 f = __ldg(p + u);
      const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int idx = 4 * u + w;  // coefficient idx / 3, channel idx % 3
        acc[idx % 3] = fmaf(b[idx / 3], fv[w], acc[idx % 3]);
      }
    }
  } else {
    // compile-time indices (a runtime-indexed b[] would live in local memory)
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      if (k < K) {
        acc[0] = fmaf(b[k], __ldg(sh + 3 * k + 0), acc[0]);
        acc[1] = fmaf(b[k], __ldg(sh + 3 * k + 1), acc[1]);
        acc[2] = fmaf(b[k], __ldg(sh + 3 * k + 2), acc[2]);
      }
    }
  }
  // np.clip(basis @ sh + 0.5, 0, None): lower clamp only
  out[0] = fmaxf(acc[0], 0.0f);
  out[1] = fmaxf(acc[1], 0.0f);
  out[2] = fmaxf(acc[2], 0.0f);
}

// k-th (0-based) set bit of a 64-bit mask
__device__ __forceinline__ int select_bit64(uint64_t m, int k) {
  uint32_t w = (uint32_t)m;
  int pos = 0;
  const int pl = __popc(w);
  if (k >= pl) {
    k -= pl;
    w = (uint32_t)(m >> 32);
    pos = 32;
  }
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    const int c = __popc(w & ((1u << s) - 1u));
    if (k >= c) {
      k -= c;
      w >>= s;
      pos += s;
    }
  }
  return pos;
}

// Culling geometry of one splat, staged in shared memory for the warp-level
// load-balanced tile enumeration.
struct SplatGeo {
  double mx, my, a, b, c, ia, ic, thr;
  float op;
  int rx0, rx1, ry0, ry1;
};
// x = q * w + r for 0 <= x < 2^22, 0 < w < 2^12: the float reciprocal
// estimate is within one of the quotient, one correction makes it exact
// (an integer division by a runtime w is a ~20-instruction sequence)
#ifndef STP_FDIVMOD
#define STP_FDIVMOD 1
#endif
__device__ __forceinline__ void divmod_small(int x, int w, int& q, int& r) {
#if STP_FDIVMOD
  q = __float2int_rz(((float)x + 0.5f) * __frcp_rn((float)w));
  r = x - q * w;
  if (r < 0) {
    --q;
    r += w;
  } else if (r >= w) {
    ++q;
    r -= w;
  }
#else
  q = x / w;
  r = x - q * w;
#endif
}

struct StagedGeo {
  double mx, my, a, b, c, ia, ic, thr;
  float op;
  int rx0, ry0, wx;
};

// Warp-cooperative enumeration of the coarse (splat, tile) pairs of the 32
// splats held by the warp's lanes (area = pairs of this lane's splat): every
// round gives each lane one pair, so work is balanced whatever the rect sizes
// (PAPER.md:589-599 load balancing, generalised).  fn(valid, owner, local)
// is called warp-uniformly once per round; owner = lane owning the pair,
// local = index of the pair in the owner's rect (row-major, rasterizer.py:331-332).
template <class F>
__device__ __forceinline__ void warp_expand(int area, int lane, F&& fn) {
  int incl = area;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(kFull, incl, 31);
  const int excl = incl - area;
  for (int base = 0; base < total; base += 32) {
    const int k = base + lane;
    int lo = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
      if (__shfl_sync(kFull, incl, lo + step - 1) <= k) lo += step;
    const int owner = lo < 31 ? lo : 31;
    const int local = k - __shfl_sync(kFull, excl, owner);
    fn(k < total, owner, local);
  }
}

// coarse tile rect (rasterizer.py:307-321), clamped in double first; empty
// rects come back as x0 > x1.
__device__ __forceinline__ void coarse_rect(double px, double py, double radius, int gw, int gh,
                                            int& x0, int& x1, int& y0, int& y1) {
  const double ts = (double)kTile;
  const double lo = -2.0;
  const double its = 1.0 / ts;  // exact (power of two): x / ts == x * its
  const double fx0 = fmin(fmax(floor((px - radius) * its), lo), (double)gw + 1);
  const double fy0 = fmin(fmax(floor((py - radius) * its), lo), (double)gh + 1);
  const double fx1 =
      fmin(fmax(fmax(ceil((px + radius) * its) - 1.0, floor(px * its)), lo), (double)gw + 1);
  const double fy1 =
      fmin(fmax(fmax(ceil((py + radius) * its) - 1.0, floor(py * its)), lo), (double)gh + 1);
  x0 = max((int)fx0, 0);
  y0 = max((int)fy0, 0);
  x1 = min((int)fx1, gw - 1);
  y1 = min((int)fy1, gh - 1);
  if (!(radius == radius)) {  // NaN radius: no tiles
    x0 = 1;
    x1 = 0;
  }
  if (x1 < x0 || y1 < y0) {
    x0 = 1;
    x1 = 0;
    y0 = 1;
    y1 = 0;
  }
}

// Exact-culled tile count (rasterizer.py:334-339) of the block's splats,
// load-balanced per warp, plus the survivors' positions in <= 64-tile rects
// (masks, for K3) and the projection stats.  Called by K1 and the SplatBatch
// ingest kernel with reason 0 (kept) .. 4 (out of range).
__device__ __forceinline__ void count_tiles(int reason, const SplatGeo& g, int64_t i, bool valid,
                                            const DevCfg& cfg, uint64_t* __restrict__ masks,
                                            uint32_t* __restrict__ rowlist,
                                            uint32_t* __restrict__ counts,
                                            uint8_t* __restrict__ state,
                                            unsigned long long* __restrict__ counters) {
  const int lane = threadIdx.x & 31;
  __shared__ StagedGeo s_geo[kPreThreads];
  __shared__ uint32_t s_cnt[kPreThreads];
  __shared__ unsigned long long s_mask[kPreThreads];
  const int wx = g.rx1 - g.rx0 + 1, wy = g.ry1 - g.ry0 + 1;
  const int full = (reason == 0 && wx > 0 && wy > 0) ? wx * wy : 0;
  // sparse rects over 64 tiles (exact culling) go to the row kernels
  const bool rows = cfg.exact && full > kMaskTiles && use_rows(g.a, g.b, g.c, g.thr, full);
  const int area = rows ? 0 : full;
  {
    StagedGeo& sg = s_geo[threadIdx.x];
    sg.mx = g.mx;
    sg.my = g.my;
    sg.a = g.a;
    sg.b = g.b;
    sg.c = g.c;
    sg.ia = g.ia;
    sg.ic = g.ic;
    sg.thr = g.thr;
    sg.op = g.op;
    sg.rx0 = g.rx0;
    sg.ry0 = g.ry0;
    sg.wx = wx;
    s_cnt[threadIdx.x] = 0;
    s_mask[threadIdx.x] = 0ull;
  }
  __syncwarp();
  const int wbase = threadIdx.x & ~31;
#ifdef STP_WORK_STATS_K1  // K1 pair counts (slots 10/11 are K6's mid stats otherwise)
  {
    const unsigned tot = __reduce_add_sync(kFull, (unsigned)full);
    const unsigned big = __reduce_add_sync(kFull, full > 64 ? (unsigned)full : 0u);
    if (lane == 0) {
      atomicAdd(counters + C_STAT + 10, (unsigned long long)tot);
      atomicAdd(counters + C_STAT + 11, (unsigned long long)big);
    }
  }
#endif
  warp_expand(area, lane, [&](bool v, int owner, int local) {
    bool keep = false;
    if (v) {
      const StagedGeo& o = s_geo[wbase + owner];
      int qy, rx;
      divmod_small(local, o.wx, qy, rx);
      const int tx = o.rx0 + rx, ty = o.ry0 + qy;
      double px, py;
      keep = !cfg.exact || tile_survives(o.mx, o.my, o.a, o.b, o.c, o.ia, o.ic, o.thr, o.op,
                                          cfg.eps, tx, ty, px, py);
    }
    const unsigned peers = __match_any_sync(kFull, v ? owner : 32 + lane);
    const unsigned kb = __ballot_sync(kFull, keep);
    if (v && lane == __ffs(peers) - 1 && (kb & peers)) {
      s_cnt[wbase + owner] += __popc(kb & peers);
      // survivors' rect positions (consecutive locals of this round) for K3
      if (local < 64) {
        const unsigned first = __ffs(peers) - 1;
        const unsigned long long bits = (unsigned long long)((kb & peers) >> first) << local;
        s_mask[wbase + owner] |= bits;
      }
    }
    __syncwarp();
  });
  // large rects: appended to the row list; k_rows_count counts them
  {
    const unsigned rb = __ballot_sync(kFull, rows);
    if (rb) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(counters + C_ROWS, (unsigned long long)__popc(rb));
      base = __shfl_sync(kFull, base, 0);
      if (rows) rowlist[base + __popc(rb & ((1u << lane) - 1))] = (uint32_t)i;
    }
  }
  const uint32_t cnt = s_cnt[threadIdx.x];
  if (valid) {
    counts[i] = cnt;
    // (rects over 64 tiles keep no survivor mask: 0, or the listed marker)
    if (cnt) masks[i] = full <= kMaskTiles ? s_mask[threadIdx.x] : 0ull;
    else if (rows) masks[i] = kRowsListed;  // K3 leaves it to k_rows_dup
    if (state) state[i] = (uint8_t)reason;
  }
  // projection stats: per-warp ballots added to per-SM slots (no block
  // barrier: warps leave the load-balanced count loop at different times)
  {
    const unsigned b1 = __ballot_sync(kFull, reason == 1), b2 = __ballot_sync(kFull, reason == 2);
    const unsigned b3 = __ballot_sync(kFull, reason == 3), b0 = __ballot_sync(kFull, reason == 0);
    if (lane == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      unsigned long long* ps = counters + C_PSTAT + (smid & 255) * 4;
      if (b1) atomicAdd(ps + 0, (unsigned long long)__popc(b1));
      if (b2) atomicAdd(ps + 1, (unsigned long long)__popc(b2));
      if (b3) atomicAdd(ps + 2, (unsigned long long)__popc(b3));
      if (b0) atomicAdd(ps + 3, (unsigned long long)__popc(b0));
    }
  }
}

__global__ void __launch_bounds__(kPreThreads, STP_K1_MINB) k_preprocess(
    StpScene sc, DevCam cam, DevCfg cfg, int gw, int gh, SplatRec* __restrict__ recs,
    uint64_t* __restrict__ masks,
    uint32_t* __restrict__ rowlist, double2* __restrict__ aux, uint32_t* __restrict__ counts,
    uint8_t* __restrict__ state,
    unsigned long long* __restrict__ counters) {
  const int64_t i = (int64_t)blockIdx.x * kPreThreads + threadIdx.x;
  const bool valid = i < sc.n;
  int reason = 4;  // 0 kept, 1 behind, 2 guard, 3 degenerate, 4 out of range
  SplatGeo g;
  g.rx0 = 1;
  g.rx1 = 0;
  g.ry0 = 1;
  g.ry1 = 0;
  g.mx = g.my = g.a = g.b = g.c = g.ia = g.ic = g.thr = 0.0;
  g.op = 0.f;

  if (valid) {
    const double* W = cam.R;
#if STP_K1_V2 && STP_K1_HOIST
    // issue every per-Gaussian input load up front (before the near-plane and
    // guard tests), so their latencies overlap instead of following the
    // projection math; culled Gaussians cost 32 B of extra reads
    float4 qf_h;
    float s0_h, s1_h, s2_h, op_h;
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(qf_h.x), "=f"(qf_h.y), "=f"(qf_h.z), "=f"(qf_h.w)
                 : "l"(reinterpret_cast<const float4*>(sc.quats) + i));
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(s0_h) : "l"(sc.scales + 3 * i + 0));
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(s1_h) : "l"(sc.scales + 3 * i + 1));
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(s2_h) : "l"(sc.scales + 3 * i + 2));
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(op_h) : "l"(sc.opacity + i));
#endif
    const double rel0 = (double)__ldg(sc.means + 3 * i + 0) - cam.pos[0];
    const double rel1 = (double)__ldg(sc.means + 3 * i + 1) - cam.pos[1];
    const double rel2 = (double)__ldg(sc.means + 3 * i + 2) - cam.pos[2];
    // p_view = rel @ W^T (gaussian_math.py:360-362)
    const double pv0 = rel0 * W[0] + rel1 * W[1] + rel2 * W[2];
    const double pv1 = rel0 * W[3] + rel1 * W[4] + rel2 * W[5];
    const double z = rel0 * W[6] + rel1 * W[7] + rel2 * W[8];
    if (!(z > cfg.near_plane)) {
      reason = 1;  // :364
    } else {
      // divisions below: fdiv (MUFU + Newton, <= 1 ulp) in the reference's
      // operation order, instead of the long IEEE division sequence
      const double px = fdiv(cam.fx * pv0, z) + cam.cx;  // :368-369
      const double py = fdiv(cam.fy * pv1, z) + cam.cy;
      const bool in_guard = (fabs(px - cam.cx) <= cfg.guard * cam.W / 2.0) &&
                            (fabs(py - cam.cy) <= cfg.guard * cam.H / 2.0);
      if (!in_guard) {
        reason = 2;  // :370-373
      } else {
#if !STP_SPLIT_SH
        // the SH row (192 B at degree 3) is only needed at the end: start
        // pulling it into L2 now, under the covariance math
        {
          const char* shp = reinterpret_cast<const char*>(sc.sh + i * sc.sh_coeffs * 3);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(shp));
          if (sc.sh_coeffs > 5) asm volatile("prefetch.global.L2 [%0];" ::"l"(shp + 128));
        }
#endif
#if STP_K1_V2 && STP_K1_SH_EARLY
        // SH colour first (gaussian_math.py:415-419), so its 48 registers of
        // coefficients are dead before the covariance algebra; opacity and
        // colour go out in one 128-bit store (a degenerate Gaussian's record
        // is never read)
        {
          const double dist = sqrt(rel0 * rel0 + rel1 * rel1 + rel2 * rel2);
          float col[3];
          sh_color(sc.sh + (int64_t)i * sc.sh_coeffs * 3, sc.sh_coeffs, (float)(rel0 / dist),
                   (float)(rel1 / dist), (float)(rel2 / dist), col);
          st128f(&recs[i].op, op_h, col[0], col[1], col[2]);
        }
#endif
#if STP_K1_V2
        // Register-lean form of the same algebra (round 2): with V = W R
        // (3 x 3), cov2 = J W R S^2 R^T W^T J^T = (J V) S^2 (J V)^T and the
        // camera-space inverse covariance M' = W inv3 W^T = V S^-2 V^T
        // (clamped 1/s), so neither cov3 nor inv3 is materialised and every
        // symmetric matrix keeps 3 or 6 values.  The record is written in
        // four 256-bit stores as soon as each part is known, instead of one
        // 160-B struct store that kept all 20 fields live to the end (K1 had
        // spilled 176 B per thread).  Same real numbers as the reference's
        // (gaussian_math.py:361-413), different rounding order (~1e-16).
        double V[9];
        {
          // _quats_to_matrices (gaussian_math.py:102-115)
#if STP_K1_HOIST
          const float4 qf = qf_h;
#else
          const float4 qf = __ldg(reinterpret_cast<const float4*>(sc.quats) + i);
#endif
          const double qw0 = qf.x, qx0 = qf.y, qy0 = qf.z, qz0 = qf.w;
          const double qn = sqrt(qw0 * qw0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0);
          const double w = fdiv(qw0, qn), x = fdiv(qx0, qn), y = fdiv(qy0, qn),
                       zq = fdiv(qz0, qn);
          const double rot[9] = {1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq),
                                 2 * (x * zq + w * y),      2 * (x * y + w * zq),
                                 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x),
                                 2 * (x * zq - w * y),      2 * (y * zq + w * x),
                                 1 - 2 * (x * x + y * y)};
#pragma unroll
          for (int aa = 0; aa < 3; ++aa)
#pragma unroll
            for (int bb = 0; bb < 3; ++bb)
              V[aa * 3 + bb] = W[aa * 3 + 0] * rot[0 * 3 + bb] + W[aa * 3 + 1] * rot[1 * 3 + bb] +
                               W[aa * 3 + 2] * rot[2 * 3 + bb];
        }
#if STP_K1_HOIST
        const double s0 = s0_h, s1 = s1_h, s2 = s2_h;
#else
        const double s0 = __ldg(sc.scales + 3 * i + 0);
        const double s1 = __ldg(sc.scales + 3 * i + 1);
        const double s2 = __ldg(sc.scales + 3 * i + 2);
#endif
        // J (gaussian_math.py:378-383): rows (J00, 0, J02), (0, J11, J12)
        const double zz = z * z;
        const double J00 = fdiv(cam.fx, z), J02 = -fdiv(cam.fx * pv0, zz);
        const double J11 = fdiv(cam.fy, z), J12 = -fdiv(cam.fy * pv1, zz);
        double a = cfg.dilation, b = 0.0, c = cfg.dilation;  // :385-387
        {
          const double ss[3] = {s0 * s0, s1 * s1, s2 * s2};
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) {
            const double B0 = J00 * V[0 * 3 + bb] + J02 * V[2 * 3 + bb];
            const double B1 = J11 * V[1 * 3 + bb] + J12 * V[2 * 3 + bb];
            a += ss[bb] * B0 * B0;
            b += ss[bb] * B0 * B1;
            c += ss[bb] * B1 * B1;
          }
        }
        const double det = a * c - b * b;
        if (!(det > 0.0)) {
          reason = 3;  // :388-390
        } else {
          reason = 0;
          SplatRec* rp = recs + i;
          const double ca = fdiv(c, det), cb = -fdiv(b, det), cc = fdiv(a, det);  // conic (:397)
          st256(&rp->mx, px, py, ca, cb);
          const double inv_a = fdiv(1.0, ca), inv_c = fdiv(1.0, cc);
          // opacity-aware radius (:399-404)
#if STP_K1_HOIST
          const float opf = op_h;
#else
          const float opf = __ldg(sc.opacity + i);
#endif
          const double op = opf;
          const double mid = 0.5 * (a + c);
          const double lam_max = mid + sqrt(fmax(mid * mid - a * c + b * b, 0.0));
          const double lg = log(op / cfg.eps);
          const double cutoff = (op > cfg.eps) ? sqrt(2.0 * lg) : 0.0;
          const double radius = cutoff * sqrt(lam_max);
          const double thr = (op > 0.0) ? lg : -INFINITY;
          int x0, x1, y0, y1;
          coarse_rect(px, py, radius, gw, gh, x0, x1, y0, y1);
          {
            const unsigned lo = ((unsigned)(uint16_t)(int16_t)x0) | ((unsigned)(uint16_t)(int16_t)x1 << 16);
            const unsigned hi = ((unsigned)(uint16_t)(int16_t)y0) | ((unsigned)(uint16_t)(int16_t)y1 << 16);
            st256(&rp->inv_a, inv_a, inv_c, thr, __hiloint2double((int)hi, (int)lo));
          }
          // M' = V diag(min(1/s, clamp)^2) V^T (:406-412) and q' = M' p_view (:413)
          {
            double is[3];
            is[0] = fmin(fdiv(1.0, s0), cfg.clamp);
            is[1] = fmin(fdiv(1.0, s1), cfg.clamp);
            is[2] = fmin(fdiv(1.0, s2), cfg.clamp);
            double m00 = 0.0, m11 = 0.0, m22 = 0.0, m01 = 0.0, m02 = 0.0, m12 = 0.0;
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) {
              const double w2 = is[bb] * is[bb];
              const double v0 = V[0 * 3 + bb], v1 = V[1 * 3 + bb], v2 = V[2 * 3 + bb];
              m00 += w2 * v0 * v0;
              m11 += w2 * v1 * v1;
              m22 += w2 * v2 * v2;
              m01 += w2 * v0 * v1;
              m02 += w2 * v0 * v2;
              m12 += w2 * v1 * v2;
            }
            const double q0 = m00 * pv0 + m01 * pv1 + m02 * z;
            const double q1 = m01 * pv0 + m11 * pv1 + m12 * z;
            const double q2 = m02 * pv0 + m12 * pv1 + m22 * z;
            st256(&rp->cc, cc, q2, m00, m11);
            st256(&rp->m[2], m22, 2.0 * m01, 2.0 * m02, 2.0 * m12);
#if STP_K1_SH_EARLY
            st128d(&rp->q0, q0, q1);
            // GlobalZ: view z and |mean - origin| (gaussian_math.py:421-430)
            if (aux) aux[i] = make_double2(z, sqrt(rel0 * rel0 + rel1 * rel1 + rel2 * rel2));
#else
            // SH colour along (mean - origin) / |mean - origin| (:415-419)
            const double dist = sqrt(rel0 * rel0 + rel1 * rel1 + rel2 * rel2);
            float col[3];
            sh_color(sc.sh + (int64_t)i * sc.sh_coeffs * 3, sc.sh_coeffs, (float)(rel0 / dist),
                     (float)(rel1 / dist), (float)(rel2 / dist), col);
            st256(&rp->q0, q0, q1,
                  __hiloint2double(__float_as_int(col[0]), __float_as_int(opf)),
                  __hiloint2double(__float_as_int(col[2]), __float_as_int(col[1])));
            // GlobalZ: view z and |mean - origin| (gaussian_math.py:421-430)
            if (aux) aux[i] = make_double2(z, dist);
#endif
          }
          g.mx = px;
          g.my = py;
          g.a = ca;
          g.b = cb;
          g.c = cc;
          g.ia = inv_a;
          g.ic = inv_c;
          g.thr = thr;
          g.op = opf;
          g.rx0 = x0;
          g.rx1 = x1;
          g.ry0 = y0;
          g.ry1 = y1;
        }
#else
        // _quats_to_matrices (gaussian_math.py:102-115)
        const float4 qf = __ldg(reinterpret_cast<const float4*>(sc.quats) + i);
        const double qw0 = qf.x, qx0 = qf.y, qy0 = qf.z, qz0 = qf.w;
        const double qn = sqrt(qw0 * qw0 + qx0 * qx0 + qy0 * qy0 + qz0 * qz0);
        const double w = fdiv(qw0, qn), x = fdiv(qx0, qn), y = fdiv(qy0, qn), zq = fdiv(qz0, qn);
        double rot[9] = {1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y),
                         2 * (x * y + w * zq),      1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x),
                         2 * (x * zq - w * y),      2 * (y * zq + w * x),  1 - 2 * (x * x + y * y)};
        const double s0 = __ldg(sc.scales + 3 * i + 0);
        const double s1 = __ldg(sc.scales + 3 * i + 1);
        const double s2 = __ldg(sc.scales + 3 * i + 2);
        const double ss[3] = {s0 * s0, s1 * s1, s2 * s2};
        double cov3[9];
#pragma unroll
        for (int aa = 0; aa < 3; ++aa)
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) {
            double acc = 0.0;
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) acc += rot[aa * 3 + bb] * ss[bb] * rot[cc * 3 + bb];
            cov3[aa * 3 + cc] = acc;
          }
        // J and M = J W (gaussian_math.py:378-383)
        const double zz = z * z;
        const double J[6] = {fdiv(cam.fx, z), 0.0, -fdiv(cam.fx * pv0, zz),
                             0.0, fdiv(cam.fy, z), -fdiv(cam.fy * pv1, zz)};
        double M[6];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int k = 0; k < 3; ++k)
            M[r * 3 + k] = J[r * 3 + 0] * W[k] + J[r * 3 + 1] * W[3 + k] + J[r * 3 + 2] * W[6 + k];
        double cov2[4];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int l = 0; l < 2; ++l) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
              for (int k = 0; k < 3; ++k) acc += M[r * 3 + j] * cov3[j * 3 + k] * M[l * 3 + k];
            cov2[r * 2 + l] = acc;
          }
        const double a = cov2[0] + cfg.dilation;  // :385-387
        const double b = cov2[1];
        const double c = cov2[3] + cfg.dilation;
        const double det = a * c - b * b;
        if (!(det > 0.0)) {
          reason = 3;  // :388-390
        } else {
          reason = 0;
          SplatRec r;
          r.mx = px;
          r.my = py;
          r.ca = fdiv(c, det);  // conic (:397)
          r.cb = -fdiv(b, det);
          r.cc = fdiv(a, det);
          r.inv_a = fdiv(1.0, r.ca);
          r.inv_c = fdiv(1.0, r.cc);
          // opacity-aware radius (:399-404)
          const float opf = __ldg(sc.opacity + i);
          const double op = opf;
          const double mid = 0.5 * (a + c);
          const double lam_max = mid + sqrt(fmax(mid * mid - a * c + b * b, 0.0));
          const double lg = log(op / cfg.eps);
          const double cutoff = (op > cfg.eps) ? sqrt(2.0 * lg) : 0.0;
          const double radius = cutoff * sqrt(lam_max);
          r.thr = (op > 0.0) ? lg : -INFINITY;
          r.op = opf;
          // packed clamped inverse covariance (:406-412) and its centre (:413)
          double is[3];
          is[0] = fmin(fdiv(1.0, s0), cfg.clamp);
          is[1] = fmin(fdiv(1.0, s1), cfg.clamp);
          is[2] = fmin(fdiv(1.0, s2), cfg.clamp);
          is[0] *= is[0];
          is[1] *= is[1];
          is[2] *= is[2];
          double inv3[9];
#pragma unroll
          for (int aa = 0; aa < 3; ++aa)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
              double acc = 0.0;
#pragma unroll
              for (int bb = 0; bb < 3; ++bb) acc += rot[aa * 3 + bb] * is[bb] * rot[cc * 3 + bb];
              inv3[aa * 3 + cc] = acc;
            }
          // camera space: M' = W inv3 W^T, q' = M' p_view (SplatRec comment)
          double WI[9];  // W inv3
#pragma unroll
          for (int aa = 0; aa < 3; ++aa)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
              WI[aa * 3 + cc] = W[aa * 3 + 0] * inv3[0 * 3 + cc] + W[aa * 3 + 1] * inv3[1 * 3 + cc] +
                                W[aa * 3 + 2] * inv3[2 * 3 + cc];
          double Mc[9];
#pragma unroll
          for (int aa = 0; aa < 3; ++aa)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
              Mc[aa * 3 + cc] = WI[aa * 3 + 0] * W[cc * 3 + 0] + WI[aa * 3 + 1] * W[cc * 3 + 1] +
                                WI[aa * 3 + 2] * W[cc * 3 + 2];
          r.m[0] = Mc[0];
          r.m[1] = Mc[4];
          r.m[2] = Mc[8];
          r.m[3] = Mc[1] + Mc[3];
          r.m[4] = Mc[2] + Mc[6];
          r.m[5] = Mc[5] + Mc[7];
          r.q0 = Mc[0] * pv0 + Mc[1] * pv1 + Mc[2] * z;
          r.q1 = Mc[3] * pv0 + Mc[4] * pv1 + Mc[5] * z;
          r.q2 = Mc[6] * pv0 + Mc[7] * pv1 + Mc[8] * z;
#if STP_SPLIT_SH
          // SH colour: K1b (k_shade), for the splats that reach a tile
          r.c0 = r.c1 = r.c2 = 0.f;
          const float col[3] = {0.f, 0.f, 0.f};
#else
          // SH colour along (mean - origin) / |mean - origin| (:415-419)
          const double dist = sqrt(rel0 * rel0 + rel1 * rel1 + rel2 * rel2);
          float col[3];
          sh_color(sc.sh + (int64_t)i * sc.sh_coeffs * 3, sc.sh_coeffs, (float)(rel0 / dist),
                   (float)(rel1 / dist), (float)(rel2 / dist), col);
          r.c0 = col[0];
          r.c1 = col[1];
          r.c2 = col[2];
#endif
          int x0, x1, y0, y1;
          coarse_rect(px, py, radius, gw, gh, x0, x1, y0, y1);
          r.rx0 = (int16_t)x0;
          r.rx1 = (int16_t)x1;
          r.ry0 = (int16_t)y0;
          r.ry1 = (int16_t)y1;
          recs[i] = r;
          // GlobalZ: view z and |mean - origin| (gaussian_math.py:421-430)
          if (aux) aux[i] = make_double2(z, sqrt(rel0 * rel0 + rel1 * rel1 + rel2 * rel2));
          g.mx = r.mx;
          g.my = r.my;
          g.a = r.ca;
          g.b = r.cb;
          g.c = r.cc;
          g.ia = r.inv_a;
          g.ic = r.inv_c;
          g.thr = r.thr;
          g.op = r.op;
          g.rx0 = x0;
          g.rx1 = x1;
          g.ry0 = y0;
          g.ry1 = y1;
        }
#endif
      }
    }
  }

  count_tiles(reason, g, i, valid, cfg, masks, rowlist, counts, state, counters);
}

// ---------------------------------------------------------------------------
// K1b: SH colour (gaussian_math.py:152-175, 415-419) of the splats that reach
// at least one tile, as a separate streaming kernel: keeping the 192 B of SH
// coefficients out of K1 leaves K1 fewer registers and the loads here all
// in flight at full occupancy.
__global__ void __launch_bounds__(256) k_shade(StpScene sc, DevCam cam,
                                               const uint32_t* __restrict__ counts,
                                               SplatRec* __restrict__ recs) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= sc.n || counts[i] == 0) return;
  const double rel0 = (double)__ldg(sc.means + 3 * i + 0) - cam.pos[0];
  const double rel1 = (double)__ldg(sc.means + 3 * i + 1) - cam.pos[1];
  const double rel2 = (double)__ldg(sc.means + 3 * i + 2) - cam.pos[2];
  const double dist = sqrt(rel0 * rel0 + rel1 * rel1 + rel2 * rel2);
  float col[3];
  sh_color(sc.sh + i * sc.sh_coeffs * 3, sc.sh_coeffs, (float)(rel0 / dist),
           (float)(rel1 / dist), (float)(rel2 / dist), col);
  recs[i].c0 = col[0];
  recs[i].c1 = col[1];
  recs[i].c2 = col[2];
}

// ---------------------------------------------------------------------------
// SplatBatch ingest: the K1 outputs from an already-projected batch
// (rasterizer.py:616-618 skips project_scene); every batch splat is kept.
__global__ void __launch_bounds__(kPreThreads) k_ingest(
    StpSplatBatch b, DevCam cam, DevCfg cfg, int gw, int gh, SplatRec* __restrict__ recs,
    uint64_t* __restrict__ masks,
    uint32_t* __restrict__ rowlist, double2* __restrict__ aux, uint32_t* __restrict__ counts,
    uint8_t* __restrict__ state,
    unsigned long long* __restrict__ counters) {
  const int64_t i = (int64_t)blockIdx.x * kPreThreads + threadIdx.x;
  const bool valid = i < b.n;
  int reason = valid ? 0 : 4;
  SplatGeo g;
  g.rx0 = 1;
  g.rx1 = 0;
  g.ry0 = 1;
  g.ry1 = 0;
  g.mx = g.my = g.a = g.b = g.c = g.ia = g.ic = g.thr = 0.0;
  g.op = 0.f;
  if (valid) {
    SplatRec r;
    r.mx = b.mean2d[2 * i];
    r.my = b.mean2d[2 * i + 1];
    r.ca = b.conic[3 * i];
    r.cb = b.conic[3 * i + 1];
    r.cc = b.conic[3 * i + 2];
    r.inv_a = 1.0 / r.ca;
    r.inv_c = 1.0 / r.cc;
    const double op = b.opacity[i];
    r.thr = (op > 0.0) ? log(op / cfg.eps) : -INFINITY;
    r.op = (float)op;
    {
      // world inverse covariance / centre -> camera space (SplatRec comment)
      const double* W = cam.R;
      const double* m6 = b.inv_cov3 + 6 * i;
      const double M[9] = {m6[0], m6[3], m6[4], m6[3], m6[1], m6[5], m6[4], m6[5], m6[2]};
      double WM[9], Mc[9];
      for (int aa = 0; aa < 3; ++aa)
        for (int cc = 0; cc < 3; ++cc)
          WM[aa * 3 + cc] = W[aa * 3] * M[cc] + W[aa * 3 + 1] * M[3 + cc] + W[aa * 3 + 2] * M[6 + cc];
      for (int aa = 0; aa < 3; ++aa)
        for (int cc = 0; cc < 3; ++cc)
          Mc[aa * 3 + cc] =
              WM[aa * 3] * W[cc * 3] + WM[aa * 3 + 1] * W[cc * 3 + 1] + WM[aa * 3 + 2] * W[cc * 3 + 2];
      r.m[0] = Mc[0];
      r.m[1] = Mc[4];
      r.m[2] = Mc[8];
      r.m[3] = Mc[1] + Mc[3];
      r.m[4] = Mc[2] + Mc[6];
      r.m[5] = Mc[5] + Mc[7];
      const double* q = b.inv_cov_center + 3 * i;
      r.q0 = W[0] * q[0] + W[1] * q[1] + W[2] * q[2];
      r.q1 = W[3] * q[0] + W[4] * q[1] + W[5] * q[2];
      r.q2 = W[6] * q[0] + W[7] * q[1] + W[8] * q[2];
    }
    r.c0 = (float)b.color[3 * i];
    r.c1 = (float)b.color[3 * i + 1];
    r.c2 = (float)b.color[3 * i + 2];
    int x0, x1, y0, y1;
    coarse_rect(r.mx, r.my, b.radius[i], gw, gh, x0, x1, y0, y1);
    r.rx0 = (int16_t)x0;
    r.rx1 = (int16_t)x1;
    r.ry0 = (int16_t)y0;
    r.ry1 = (int16_t)y1;
    recs[i] = r;
    if (aux)
      aux[i] = make_double2(b.global_depth ? b.global_depth[i] : 0.0,
                            b.center_dist ? b.center_dist[i] : 0.0);
    g.mx = r.mx;
    g.my = r.my;
    g.a = r.ca;
    g.b = r.cb;
    g.c = r.cc;
    g.ia = r.inv_a;
    g.ic = r.inv_c;
    g.thr = r.thr;
    g.op = r.op;
    g.rx0 = x0;
    g.rx1 = x1;
    g.ry0 = y0;
    g.ry1 = y1;
  }
  count_tiles(reason, g, i, valid, cfg, masks, rowlist, counts, state, counters);
}

// ---------------------------------------------------------------------------
// K2 exclusive scan of per-splat tile counts (three phases, 4096 per block).

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
static_assert(kScanTile == kScanBlockItems, "the workspace sizes the K2 partials by kScanBlockItems");

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t s = (lane < (int)(blockDim.x >> 5)) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    s_warp[lane] = s;
  }
  __syncthreads();
  total = s_warp[(blockDim.x >> 5) - 1];
  const uint32_t warp_off = w ? s_warp[w - 1] : 0;
  __syncthreads();
  return warp_off + x - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_partials(const uint32_t* __restrict__ counts,
                                                                int64_t n, uint32_t* partials) {
  __shared__ uint32_t s_warp[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t sum = 0;
  if (base + kScanItems <= n) {
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      const uint4 c = *reinterpret_cast<const uint4*>(counts + base + 4 * q);
      sum += c.x + c.y + c.z + c.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (base + k < n) sum += counts[base + k];
  }
  uint32_t total;
  block_excl_scan(sum, s_warp, total);
  if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_top(uint32_t* partials, int nb,
                                                   unsigned long long* counters) {
  __shared__ uint32_t s_warp[32];
  unsigned long long carry = 0;
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const uint32_t v = (i < nb) ? partials[i] : 0;
    uint32_t total;
    const uint32_t ex = block_excl_scan(v, s_warp, total);
    if (i < nb) partials[i] = (uint32_t)(carry + ex);
    carry += total;
  }
  if (threadIdx.x == 0) counters[C_ENTRIES] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_final(const uint32_t* __restrict__ counts,
                                                             int64_t n,
                                                             const uint32_t* __restrict__ partials,
                                                             uint32_t* __restrict__ offsets) {
  __shared__ uint32_t s_warp[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t sum = 0;
  // a thread's 16 counts are one 64-B run: 128-bit loads and stores where
  // the run is whole (the arrays are 16-B aligned)
  const bool whole = base + kScanItems <= n;
  if (whole) {
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q) {
      const uint4 c = *reinterpret_cast<const uint4*>(counts + base + 4 * q);
      v[4 * q] = c.x;
      v[4 * q + 1] = c.y;
      v[4 * q + 2] = c.z;
      v[4 * q + 3] = c.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = (base + k < n) ? counts[base + k] : 0;
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) sum += v[k];
  uint32_t total;
  uint32_t run = block_excl_scan(sum, s_warp, total) + partials[blockIdx.x];
  uint32_t o[kScanItems];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    o[k] = run;
    run += v[k];
  }
  if (whole) {
#pragma unroll
    for (int q = 0; q < kScanItems / 4; ++q)
      *reinterpret_cast<uint4*>(offsets + base + 4 * q) =
          make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (base + k < n) offsets[base + k] = o[k];
  }
}

// ---------------------------------------------------------------------------
// K3 duplicate.

#ifndef STP_K3_PREFETCH
#define STP_K3_PREFETCH 0  // K3 0.1336 -> 0.1309 ms but the step 4.279 -> 4.288 ms (profiles/r2ax): off
#endif
// GZ: GlobalZ keys (view z from aux) -- a template parameter so the
// hierarchical instantiation carries no GlobalZ code
template <bool GZ>
__global__ void __launch_bounds__(kPreThreads) k_duplicate(
    const SplatRec* __restrict__ recs, const uint64_t* __restrict__ masks,
    const uint32_t* __restrict__ counts,
    const uint32_t* __restrict__ offsets, int64_t n, DevCam cam, DevCfg cfg, int gw,
    int depth_bits, int id_bits, int64_t ecap, const double2* __restrict__ aux,
    uint64_t* __restrict__ keys) {
  __shared__ uint32_t s_pos[kPreThreads];
  __shared__ unsigned long long s_m[kPreThreads];
  const int64_t i = (int64_t)blockIdx.x * kPreThreads + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const uint32_t cnt = (i < n) ? counts[i] : 0;
  int area = 0;
  if (cnt > 0) {
#if STP_K3_PREFETCH
    // the warp_expand rounds below read this record's two lines once per
    // owner round: start pulling them into L2 now
    asm volatile("prefetch.global.L2 [%0];" ::"l"(recs + i));
#endif
    const short4 rc = *reinterpret_cast<const short4*>(&recs[i].rx0);
    area = (rc.y - rc.x + 1) * (rc.w - rc.z + 1);
    // rects of <= 64 tiles: K1 left the survivors' positions in a mask, so
    // only surviving pairs are enumerated (no second cull); larger ones go
    // row by row below (exact culling)
    s_m[threadIdx.x] = masks[i];
    if (area <= kMaskTiles) area = (int)cnt;
    else if (s_m[threadIdx.x] == kRowsListed) area = 0;  // k_rows_dup
    s_pos[threadIdx.x] = offsets[i];
  }
  __syncwarp();
  const int wbase = threadIdx.x & ~31;
  const unsigned lt_mask = (1u << lane) - 1;
  warp_expand(area, lane, [&](bool v, int owner, int local) {
    // the owner's record straight from L1/L2 (lanes of one owner broadcast),
    // in 256-bit loads: the culling line now, the t_opt fields for survivors
    const int64_t gid = (int64_t)blockIdx.x * kPreThreads + wbase + owner;
    const SplatRec* rp = recs + gid;
    bool keep = false;
    int tx = 0, ty = 0;
    double ptx = 0.0, pty = 0.0;
    double mx = 0.0, my = 0.0;
    if (v) {
      double ca, cb, ia, ic, thr, rectd;
      ld256(&rp->mx, mx, my, ca, cb);
      ld256(&rp->inv_a, ia, ic, thr, rectd);
      const double cc = __ldg(&rp->cc);
      const unsigned rlo = (unsigned)__double2loint(rectd), rhi = (unsigned)__double2hiint(rectd);
      const int rx0 = (int16_t)(rlo & 0xffffu), rx1 = (int16_t)(rlo >> 16);
      const int ry0 = (int16_t)(rhi & 0xffffu), ry1 = (int16_t)(rhi >> 16);
      const int w = rx1 - rx0 + 1;
      if (w * (ry1 - ry0 + 1) <= 64) {
        const int b = select_bit64(s_m[wbase + owner], local);
        int qy, rx;
        divmod_small(b, w, qy, rx);
        tx = rx0 + rx;
        ty = ry0 + qy;
        if (!GZ)  // the peak only feeds the t_opt key
          max_point(mx, my, ca, cb, cc, ia, ic, (double)(tx * kTile), (double)(ty * kTile), 16.0,
                    0.0625, ptx, pty);
        keep = true;
      } else {
        int qy, rx;
        divmod_small(local, w, qy, rx);
        tx = rx0 + rx;
        ty = ry0 + qy;
        keep = tile_survives(mx, my, ca, cb, cc, ia, ic, thr, __ldg(&rp->op), cfg.eps, tx, ty,
                             ptx, pty);
        if (!cfg.exact) keep = true;
      }
    }
    // deterministic slot: rank among this round's survivors of the same splat
    const unsigned peers = __match_any_sync(kFull, v ? owner : 32 + lane);
    const unsigned kb = __ballot_sync(kFull, keep) & peers;
    const uint32_t base = v ? s_pos[wbase + owner] : 0;
    __syncwarp();
    if (keep) {
      // rasterizer.py:343-350: view z (GlobalZ) or t_opt at the 16x16 peak
      double depth;
      if (GZ) {
        depth = aux[gid].x;
      } else {
        double cc, q2, q0, q1, x0, x1;
        double mm[6];
        ld256(&rp->cc, cc, q2, mm[0], mm[1]);
        ld256(&rp->m[2], mm[2], mm[3], mm[4], mm[5]);
        ld256(&rp->q0, q0, q1, x0, x1);
        double u, wv, vn;
        cam_ray(cam, ptx, pty, u, wv, vn);
        depth = key_rec(mm, q0, q1, q2, u, wv, vn);
      }
      const uint32_t pos = base + __popc(kb & lt_mask);
      if ((int64_t)pos < ecap) {
        const uint64_t key = ((uint64_t)(uint32_t)(ty * gw + tx) << depth_bits) |
                             (depth_key(depth) >> (32 - depth_bits));
        keys[pos] = (key << id_bits) | (uint64_t)gid;
      }
    }
    if (v && lane == __ffs(peers) - 1 && kb) s_pos[wbase + owner] = base + __popc(kb);
    __syncwarp();
  });
}

// ---------------------------------------------------------------------------
// Sparse large rects (K1b count, K3b duplicate).  A Gaussian whose coarse
// rect exceeds kMaskTiles tiles and is mostly empty (use_rows: long thin or
// faint splats; up to thousands of tiles at 4K, most far from the ellipse)
// is listed by K1 and handled here instead of tile by tile: one warp per
// (Gaussian, 32-row chunk) unit, the chunk's rows one per lane, each row's
// candidate columns from row_span, and only those candidates take the exact
// test (tile_survives), spread over the lanes by warp_expand.  Same survivors
// as testing every tile.

template <class F>
__device__ __forceinline__ void for_row_tiles(const SplatRec& o, int r0, int nrows, double eps,
                                              F&& fn) {
  const int lane = threadIdx.x & 31;
  int lo = 1, hi = 0;
  const int ty = o.ry0 + r0 + lane;
  const bool v = lane < nrows;
  if (v) row_span(o.mx, o.my, o.ca, o.cb, o.cc, o.thr, ty, o.rx0, o.rx1, lo, hi);
  warp_expand(v && hi >= lo ? hi - lo + 1 : 0, lane, [&](bool v2, int u, int col) {
    const int tyu = __shfl_sync(kFull, ty, u);
    const int tx = __shfl_sync(kFull, lo, u) + col;
    bool keep = false;
    double ptx = 0.0, pty = 0.0;
    if (v2)
      keep = tile_survives(o.mx, o.my, o.ca, o.cb, o.cc, o.inv_a, o.inv_c, o.thr, o.op, eps, tx,
                           tyu, ptx, pty);
    fn(keep, tx, tyu, ptx, pty);
  });
}

// unit w -> (listed Gaussian, rows [r0, r0 + nr)); cpg = 32-row chunks per
// Gaussian (ceil(grid_h / 32)), the surplus chunks of shorter rects are empty
__device__ __forceinline__ const SplatRec& row_unit(const SplatRec* __restrict__ recs,
                                                    const uint32_t* __restrict__ rowlist,
                                                    int64_t w, int cpg, uint32_t& id, int& r0,
                                                    int& nr) {
  id = rowlist[w / cpg];
  const SplatRec& o = recs[id];
  r0 = (int)(w % cpg) * 32;
  nr = max(0, min(o.ry1 - o.ry0 + 1 - r0, 32));
  return o;
}

__global__ void __launch_bounds__(256) k_rows_count(const SplatRec* __restrict__ recs,
                                                    const uint32_t* __restrict__ rowlist,
                                                    const unsigned long long* counters,
                                                    DevCfg cfg, int cpg,
                                                    uint32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t units = (int64_t)counters[C_ROWS] * cpg;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < units;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    uint32_t id;
    int r0, nr;
    const SplatRec& o = row_unit(recs, rowlist, w, cpg, id, r0, nr);
    if (nr == 0) continue;
    unsigned cnt = 0;
    for_row_tiles(o, r0, nr, cfg.eps, [&](bool keep, int, int, double, double) {
      cnt += __popc(__ballot_sync(kFull, keep));
    });
    // counts[id] is 0 from K1; the chunks of one Gaussian add up
    if (lane == 0 && cnt) atomicAdd(counts + id, cnt);
  }
}

__global__ void __launch_bounds__(256) k_rows_dup(const SplatRec* __restrict__ recs,
                                                  const uint32_t* __restrict__ rowlist,
                                                  const unsigned long long* counters,
                                                  uint32_t* __restrict__ offsets, DevCam cam,
                                                  DevCfg cfg, int cpg, int gw, int depth_bits,
                                                  int id_bits, int64_t ecap,
                                                  const double2* __restrict__ aux,
                                                  uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1;
  const int64_t units = (int64_t)counters[C_ROWS] * cpg;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < units;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    uint32_t id;
    int r0, nr;
    const SplatRec& o = row_unit(recs, rowlist, w, cpg, id, r0, nr);
    if (nr == 0) continue;
    for_row_tiles(o, r0, nr, cfg.eps, [&](bool keep, int tx, int ty, double ptx, double pty) {
      // slots: the Gaussian's offset is its write cursor (its entries are
      // distinct sort words, so their order in the unsorted array is free)
      const unsigned kb = __ballot_sync(kFull, keep);
      uint32_t base = 0;
      if (lane == 0 && kb) base = atomicAdd(offsets + id, (uint32_t)__popc(kb));
      base = __shfl_sync(kFull, base, 0);
      if (keep) {
        const double depth = aux ? aux[id].x : key_rec_at(cam, o, ptx, pty);  // :343-350
        const uint32_t p = base + __popc(kb & lt_mask);
        if ((int64_t)p < ecap) {
          const uint64_t key = ((uint64_t)(uint32_t)(ty * gw + tx) << depth_bits) |
                               (depth_key(depth) >> (32 - depth_bits));
          keys[p] = (key << id_bits) | (uint64_t)id;
        }
      }
    });
  }
}

// ---------------------------------------------------------------------------
// launchers

void launch_init(const Frame& f, cudaStream_t s) {
  // epoch tags of the onesweep look-back (never cleared): unique per frame in
  // the process, never 0 (0 reads as "not published")
  static std::atomic<unsigned long long> g_epoch{0};
  unsigned long long ep = ++g_epoch & 0xffffffffull;
  if (ep == 0) ep = ++g_epoch & 0xffffffffull;
  const int hist_n = f.passes * 256;
  const int work = max(max(hist_n, f.n_tiles), (int)C_COUNT);
  const int blocks = min((work + 255) / 256, 1024);
  k_init<<<blocks, 256, 0, s>>>(f.counters, f.hist, hist_n, f.ranges, f.n_tiles, f.cam, f.camp,
                                ep);
}

// grid of the row-culling kernels: the list length is on the device, so a
// fixed grid of warps strides over it (idle warps exit at once)
static unsigned rows_blocks(const Frame& f) {
  const int64_t b = (f.n + 255) / 256;
  const int64_t cap = (int64_t)device_sm_count() * 8;
  return (unsigned)(b < cap ? b : cap);
}

static void launch_rows_count(const Frame& f, cudaStream_t s) {
  if (f.cfg.exact)
    k_rows_count<<<rows_blocks(f), 256, 0, s>>>(f.recs, f.rowlist, f.counters, f.cfg,
                                                (f.gh + 31) / 32, f.counts);
}

void launch_preprocess(const Frame& f, const StpScene& sc, cudaStream_t s) {
  if (f.n == 0) return;
  const int64_t blocks = (f.n + kPreThreads - 1) / kPreThreads;
  k_preprocess<<<(unsigned)blocks, kPreThreads, 0, s>>>(sc, f.cam, f.cfg, f.gw, f.gh, f.recs,
                                                      f.masks,
                                                      f.rowlist, f.globalz ? f.aux : nullptr,
                                                      f.counts, f.state, f.counters);
#if STP_SPLIT_SH
  k_shade<<<(unsigned)blocks, 256, 0, s>>>(sc, f.cam, f.counts, f.recs);
#endif
  launch_rows_count(f, s);
}

// K1c (float64 outputs only): the SH colour of every kept Gaussian in
// float64, sh_basis (gaussian_math.py:152-175) and the clipped einsum
// (:415-419) as the reference evaluates them; blended by the XM_F64 K6
// instead of the float32 record colour.
__global__ void __launch_bounds__(256) k_shade64(StpScene sc, DevCam cam,
                                                 const uint8_t* __restrict__ state,
                                                 double* __restrict__ col) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= sc.n || state[i] != 0) return;
  const double r0 = (double)sc.means[3 * i + 0] - cam.pos[0];
  const double r1 = (double)sc.means[3 * i + 1] - cam.pos[1];
  const double r2 = (double)sc.means[3 * i + 2] - cam.pos[2];
  const double dist = sqrt(r0 * r0 + r1 * r1 + r2 * r2);
  const double x = r0 / dist, y = r1 / dist, z = r2 / dist;
  const double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  const double b[16] = {c_SH_C0,
                        -c_SH_C1 * y,
                        c_SH_C1 * z,
                        -c_SH_C1 * x,
                        c_SH_C2[0] * xy,
                        c_SH_C2[1] * yz,
                        c_SH_C2[2] * (2.0 * zz - xx - yy),
                        c_SH_C2[3] * xz,
                        c_SH_C2[4] * (xx - yy),
                        c_SH_C3[0] * y * (3.0 * xx - yy),
                        c_SH_C3[1] * xy * z,
                        c_SH_C3[2] * y * (4.0 * zz - xx - yy),
                        c_SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
                        c_SH_C3[4] * x * (4.0 * zz - xx - yy),
                        c_SH_C3[5] * z * (xx - yy),
                        c_SH_C3[6] * x * (xx - 3.0 * yy)};
  const float* sh = sc.sh + i * sc.sh_coeffs * 3;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < sc.sh_coeffs; ++k)
    for (int c = 0; c < 3; ++c) acc[c] += b[k] * (double)sh[3 * k + c];
  for (int c = 0; c < 3; ++c) col[3 * i + c] = fmax(acc[c] + 0.5, 0.0);
}

void launch_shade64(const Frame& f, const StpScene& sc, double* col64, cudaStream_t s) {
  if (f.n == 0) return;
  k_shade64<<<(unsigned)((f.n + 255) / 256), 256, 0, s>>>(sc, f.cam, f.state, col64);
}

void launch_ingest(const Frame& f, const StpSplatBatch& b, cudaStream_t s) {
  if (f.n == 0) return;
  const int64_t blocks = (f.n + kPreThreads - 1) / kPreThreads;
  k_ingest<<<(unsigned)blocks, kPreThreads, 0, s>>>(b, f.cam, f.cfg, f.gw, f.gh, f.recs,
                                                  f.masks,
                                                  f.rowlist, f.globalz ? f.aux : nullptr,
                                                  f.counts, f.state, f.counters);
  launch_rows_count(f, s);
}

void launch_scan(const Frame& f, cudaStream_t s) {
  if (f.n == 0) return;
  const int nb = (int)((f.n + kScanTile - 1) / kScanTile);
  k_scan_partials<<<nb, kScanThreads, 0, s>>>(f.counts, f.n, f.scan_scratch);
  k_scan_top<<<1, 1024, 0, s>>>(f.scan_scratch, nb, f.counters);
  k_scan_final<<<nb, kScanThreads, 0, s>>>(f.counts, f.n, f.scan_scratch, f.offsets);
}

void launch_duplicate(const Frame& f, cudaStream_t s) {
  if (f.n == 0) return;
  const int64_t blocks = (f.n + kPreThreads - 1) / kPreThreads;
  (f.globalz ? k_duplicate<true> : k_duplicate<false>)<<<(unsigned)blocks, kPreThreads, 0, s>>>(f.recs, f.masks, f.counts, f.offsets, f.n,
                                                     f.cam,
                                                     f.cfg, f.gw, f.depth_bits, f.id_bits, f.ecap,
                                                     f.globalz ? f.aux : nullptr, f.keys[0]);
  if (f.cfg.exact)
    k_rows_dup<<<rows_blocks(f), 256, 0, s>>>(f.recs, f.rowlist, f.counters, f.offsets, f.cam,
                                              f.cfg, (f.gh + 31) / 32, f.gw, f.depth_bits, f.id_bits, f.ecap,
                                              f.globalz ? f.aux : nullptr, f.keys[0]);
}

}  // namespace stp
