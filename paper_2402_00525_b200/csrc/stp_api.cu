// C ABI (include/stp.h): workspace carve-up, config validation, the K0..K6
// launch sequence of one view, and stats read-back.
#include <cstdio>
#include <cstring>

#include <algorithm>

#include "stp_common.cuh"

namespace stp {
size_t render_smem_bytes(int qt, int qm);

namespace {

constexpr int kSortTile = kSortPartition;
constexpr size_t kAlign = 256;

size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

int tile_bits(int n_tiles) {
  int b = 0;
  while ((1 << b) < n_tiles) ++b;
  return b;
}

void plan(int64_t n, int32_t W, int32_t H, int64_t ecap, StpLayout& L) {
  memset(&L, 0, sizeof(L));
  L.grid_w = (W + kTile - 1) / kTile;
  L.grid_h = (H + kTile - 1) / kTile;
  L.n_tiles = L.grid_w * L.grid_h;
  // One 64-bit word per (tile, splat) entry:
  //   (tile << depth_bits | top depth_bits of the fp32-orderable depth) << id_bits | id
  // The sort key (tile | depth) fills whole 8-bit digits (depth >= 24 bits
  // when the word allows), so a 1080p frame sorts 40 bits in 5 passes that
  // move 8 B per entry; the id rides along in the low bits (stable LSD keeps
  // Gaussian order inside equal keys = the rank tie-break).  K5 re-orders
  // runs of equal keys by the float64 depth, which makes the truncation
  // invisible in the final order.
  {
    const int tb = tile_bits(L.n_tiles);
    int ib = 1;
    while (ib < 31 && (int64_t)1 << ib < n) ++ib;
    L.id_bits = ib;
    int kb = ((tb + 24 + 7) / 8) * 8;
    if (kb > 64 - ib) kb = 64 - ib;
    if (kb - tb > 32) kb = tb + 32;
    L.sort_bits = kb;
    L.depth_bits = kb - tb;
  }
  L.sort_passes = (L.sort_bits + 7) / 8;
  L.entry_capacity = ecap;
  L.partitions = (int32_t)((ecap + kSortTile - 1) / kSortTile);
  L.splat_record_bytes = (int32_t)sizeof(SplatRec);
  L.final_buffer = L.sort_passes & 1;
  const int64_t nb = (n + kScanBlockItems - 1) / kScanBlockItems;  // K2 partials
  size_t o = 0;
  L.counters = o;     o = align_up(o + C_COUNT * 8);
  L.hist = o;         o = align_up(o + 8 * 256 * 4);
  L.ranges = o;       o = align_up(o + (size_t)L.n_tiles * 8);
  L.scan_scratch = o; o = align_up(o + (size_t)(nb + 1) * 4);
  L.recs = o;         o = align_up(o + (size_t)n * sizeof(SplatRec));
  L.camera = o;       o = align_up(o + sizeof(DevCam));
  L.masks = o;        o = align_up(o + (size_t)n * 8);
  L.state = o;        o = align_up(o + (size_t)n);
  L.counts = o;       o = align_up(o + (size_t)n * 4);
  L.offsets = o;      o = align_up(o + (size_t)n * 4);
  L.rowlist = o;      o = align_up(o + (size_t)n * 4);
  L.aux = o;          o = align_up(o + (size_t)n * 16);
  L.lookback = o;     o = align_up(o + (size_t)L.sort_passes * L.partitions * 256 * 8);
  L.keys0 = o;        o = align_up(o + (size_t)ecap * 8);
  L.keys1 = o;        o = align_up(o + (size_t)ecap * 8);
  L.vals = o;         o = align_up(o + (size_t)ecap * 4);
  L.total = o;
}

int64_t max_capacity(int64_t n, int32_t W, int32_t H, size_t ws_bytes) {
  // per-entry bytes: 2 x 8 (keys) + 4 (ids) + lookback (passes * 256 * 8 / 4096)
  StpLayout L0;
  plan(n, W, H, 0, L0);
  if (ws_bytes < L0.total) return -1;
  // largest e with plan(e).total <= ws_bytes (monotone in e): binary search
  // from the per-entry estimate, so stp_workspace_bytes(.., e) round-trips
  const double per = 20.0 + (double)L0.sort_passes * 256 * 8 / kSortTile;
  int64_t hi = (int64_t)((double)(ws_bytes - L0.total) / per) + kSortTile + 1;
  int64_t lo = 0;
  StpLayout L;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    plan(n, W, H, mid, L);
    if (L.total <= ws_bytes) lo = mid;
    else hi = mid - 1;
  }
  int64_t e = lo;
  // look-back words hold 30-bit counts; offsets are uint32
  const int64_t lim = (1ll << 30) - 1;
  if (e > lim) e = lim;
  return e < 0 ? 0 : e;
}

const char* kErrors[] = {"ok", "invalid configuration", "data error",
                         "workspace too small for the frame's entries", "CUDA error"};

int cfg_check(const StpConfig* c) {
  if (!c) return STP_ERR_CONFIG;
  if (c->tile_size != 16) return STP_ERR_CONFIG;
  if (c->sort_mode < STP_MODE_HIERARCHICAL || c->sort_mode > STP_MODE_WINDOW)
    return STP_ERR_CONFIG;
  if (!(c->alpha_cap > 0.0 && c->alpha_cap < 1.0)) return STP_ERR_CONFIG;
  if (c->record_cap < 0) return STP_ERR_CONFIG;
  if (c->tile_end > 0 && (c->tile_begin < 0 || c->tile_begin >= c->tile_end))
    return STP_ERR_CONFIG;
  if (c->sort_mode == STP_MODE_GLOBALZ || c->sort_mode == STP_MODE_FULL) return STP_OK;
  // Window(size): validate_mode (rasterizer.py:96-98); a register window up
  // to 16, a shared-memory heap up to STP_WINDOW_MAX
  if (c->sort_mode == STP_MODE_WINDOW)
    return (c->q_head >= 1 && c->q_head <= STP_WINDOW_MAX) ? STP_OK : STP_ERR_CONFIG;
  // validate_mode (rasterizer.py:98-115)
  if (c->q_tail < 64 || c->q_tail % 32 != 0) return STP_ERR_CONFIG;
  if (c->q_mid < 4 || c->q_mid % 4 != 0) return STP_ERR_CONFIG;
  if (c->q_head < 1) return STP_ERR_CONFIG;
  if (c->b_load < 1 || c->b_load >= c->q_tail) return STP_ERR_CONFIG;
  if (c->b_mid < 1 || c->b_head < 1) return STP_ERR_CONFIG;
  if (c->b_head > c->q_mid) return STP_ERR_CONFIG;
  // RenderConfig (rasterizer.py:196-203)
  if (!(c->alpha_cap > 0.0 && c->alpha_cap < 1.0)) return STP_ERR_CONFIG;
  // B200 kernel envelope: default batches, queues that fit shared memory
  if (c->b_load != 32 || c->b_mid != 16 || c->b_head != 4) return STP_ERR_CONFIG;
  if (c->q_tail > 256 || c->q_mid > 64 || c->q_head > 16) return STP_ERR_CONFIG;
  if (c->record_cap < 0) return STP_ERR_CONFIG;
  return STP_OK;
}

bool carve_frame(int64_t n, const StpCamera* cam, const StpConfig* cfg, void* ws,
                 size_t ws_bytes, Frame& f, StpLayout& L) {
  const int64_t ecap = max_capacity(n, cam->width, cam->height, ws_bytes);
  if (ecap < 0) return false;
  plan(n, cam->width, cam->height, ecap, L);
  unsigned char* b = static_cast<unsigned char*>(ws);
  f.recs = reinterpret_cast<SplatRec*>(b + L.recs);
  f.camp = reinterpret_cast<DevCam*>(b + L.camera);
  f.masks = reinterpret_cast<uint64_t*>(b + L.masks);
  f.rowlist = reinterpret_cast<uint32_t*>(b + L.rowlist);
  f.aux = reinterpret_cast<double2*>(b + L.aux);
  f.globalz = cfg->sort_mode == STP_MODE_GLOBALZ ? 1 : 0;
  f.sort_mode = cfg->sort_mode;
  f.tile0 = 0;
  f.tile1 = L.n_tiles;
  if (cfg->tile_end > 0) {
    f.tile0 = std::max(0, std::min(cfg->tile_begin, L.n_tiles));
    f.tile1 = std::max(f.tile0, std::min(cfg->tile_end, L.n_tiles));
  }
  f.status = nullptr;
  f.col64 = nullptr;
  f.state = b + L.state;
  f.counts = reinterpret_cast<uint32_t*>(b + L.counts);
  f.offsets = reinterpret_cast<uint32_t*>(b + L.offsets);
  f.keys[0] = reinterpret_cast<uint64_t*>(b + L.keys0);
  f.keys[1] = reinterpret_cast<uint64_t*>(b + L.keys1);
  f.vals = reinterpret_cast<uint32_t*>(b + L.vals);
  f.ranges = reinterpret_cast<uint2*>(b + L.ranges);
  f.counters = reinterpret_cast<unsigned long long*>(b + L.counters);
  f.hist = reinterpret_cast<uint32_t*>(b + L.hist);
  f.lookback = reinterpret_cast<unsigned long long*>(b + L.lookback);
  f.scan_scratch = reinterpret_cast<uint32_t*>(b + L.scan_scratch);
  f.n = n;
  f.ecap = ecap;
  f.gw = L.grid_w;
  f.gh = L.grid_h;
  f.n_tiles = L.n_tiles;
  f.passes = L.sort_passes;
  f.depth_bits = L.depth_bits;
  f.id_bits = L.id_bits;
  f.partitions = L.partitions;
  memcpy(f.cam.R, cam->R, sizeof(f.cam.R));
  memcpy(f.cam.pos, cam->pos, sizeof(f.cam.pos));
  f.cam.fx = cam->fx;
  f.cam.fy = cam->fy;
  f.cam.cx = cam->cx;
  f.cam.cy = cam->cy;
  f.cam.inv_fx = 1.0 / cam->fx;
  f.cam.inv_fy = 1.0 / cam->fy;
  f.cam.W = cam->width;
  f.cam.H = cam->height;
  f.cfg.eps = cfg->eps;
  f.cfg.term = cfg->termination;
  f.cfg.cap = cfg->alpha_cap;
  for (int i = 0; i < 3; ++i) f.cfg.bg[i] = cfg->bg[i];
  f.cfg.near_plane = cfg->near_plane;
  f.cfg.guard = cfg->guard;
  f.cfg.dilation = cfg->dilation;
  f.cfg.clamp = cfg->inv_scale_clamp;
  f.cfg.q_tail = cfg->q_tail;
  f.cfg.q_mid = cfg->q_mid;
  f.cfg.q_head = cfg->q_head;
  f.cfg.mid_center = cfg->mid_depth_at_center;
  f.cfg.with_depth = cfg->with_depth;
  f.cfg.exact = cfg->exact_culling;
  f.cfg.rec_cap = cfg->record_cap;
  return true;
}

// One view.  `ev` (n_ev = 5 or 8 events, or null) is recorded at the stage
// boundaries [init+K1 | K2+K3 | K4+K5 | K6] (5) or at every kernel boundary
// [K0 | K1 | K2 | K3 | K4 | K5 | K6] (8); with `ms` the stream is synchronised
// and the 4 stage times returned.
int render_one(const StpScene* sc, const StpSplatBatch* batch, const StpCamera* cam,
               const StpConfig* cfg, void* ws, size_t ws_bytes, const StpOutputs* out,
               cudaStream_t s, cudaEvent_t* ev, int n_ev, float* ms,
               const StpGrads* grads = nullptr) {
  Frame f;
  StpLayout L;
  if (!carve_frame(batch ? batch->n : sc->n, cam, cfg, ws, ws_bytes, f, L))
    return STP_ERR_WORKSPACE_TOO_SMALL;
  if (cfg->sort_mode == STP_MODE_HIERARCHICAL &&
      (size_t)render_smem_bytes(cfg->q_tail, cfg->q_mid) > 227 * 1024)
    return STP_ERR_CONFIG;
  f.status = out->status;
  cudaEvent_t own[5];
  if (ms && !ev) {
    for (int i = 0; i < 5; ++i) cudaEventCreate(&own[i]);
    ev = own;
    n_ev = 5;
  }
  const bool fine = ev && n_ev == STP_KERNEL_EVENTS;
  // event i of the 8-event scheme; the 5-event scheme records a subset
  auto mark = [&](int k8) {
    if (!ev) return;
    if (fine) {
      cudaEventRecord(ev[k8], s);
      return;
    }
    static const int k5[8] = {0, -1, 1, -1, 2, -1, 3, 4};
    if (k5[k8] >= 0) cudaEventRecord(ev[k5[k8]], s);
  };
  mark(0);
  launch_init(f, s);
  mark(1);
  StpOutputs o = *out;
  if (o.state) f.state = o.state;
  if (batch) launch_ingest(f, *batch, s);
  else launch_preprocess(f, *sc, s);
  if (o.color64) {
    // float64 outputs: blend the float64 colour (a SplatBatch's own, or the
    // SH colour re-evaluated in float64 for the kept Gaussians)
    if (batch) f.col64 = batch->color;
    else if (o.splat_color64) {
      launch_shade64(f, *sc, o.splat_color64, s);
      f.col64 = o.splat_color64;
    }
  }
  mark(2);
  launch_scan(f, s);
  mark(3);
  launch_duplicate(f, s);
  mark(4);
  const int buf = launch_sort(f, s);
  mark(5);
  launch_ranges(f, buf, s);
  mark(6);
  if (grads) {
    // backward (gradients.py:103-162): K6 replayed twice over the same bins,
    // first for each pixel's float64 colour sum and final T, then with the
    // per-contribution gradients scattered by Gaussian id
    const int64_t n = f.n;
    if (n > 0) {
      cudaMemsetAsync(grads->d_color, 0, (size_t)n * 3 * sizeof(double), s);
      cudaMemsetAsync(grads->d_opacity, 0, (size_t)n * sizeof(double), s);
      cudaMemsetAsync(grads->d_mean2d, 0, (size_t)n * 2 * sizeof(double), s);
      cudaMemsetAsync(grads->d_conic, 0, (size_t)n * 3 * sizeof(double), s);
    }
    DevGrads g;
    g.upstream = grads->upstream;
    g.pix = grads->pix_state;
    g.d_color = grads->d_color;
    g.d_opacity = grads->d_opacity;
    g.d_mean2d = grads->d_mean2d;
    g.d_conic = grads->d_conic;
    launch_render(f, buf, o, s, XM_FWD, &g);
    // the persistent K6 hands out (tile, pair) items from frame counters and
    // per-SM rings: clear them for the second replay
    cudaMemsetAsync(f.counters + C_TILE, 0, sizeof(unsigned long long), s);
    cudaMemsetAsync(f.counters + C_SM, 0, (size_t)(C_PSTAT - C_SM) * 8, s);
    launch_render(f, buf, o, s, XM_BWD, &g);
  } else {
    launch_render(f, buf, o, s);
  }
  mark(7);
  if (ms) {
    cudaEventSynchronize(ev[4]);
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]);
    if (ev == own)
      for (int i = 0; i < 5; ++i) cudaEventDestroy(own[i]);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "stp: CUDA error %s\n", cudaGetErrorString(e));
    return STP_ERR_CUDA;
  }
  return STP_OK;
}

int fill_stats(const void* ws, size_t ws_bytes, int64_t n, int32_t W, int32_t H, StpStats* st,
               cudaStream_t s) {
  StpLayout L;
  const int64_t ecap = max_capacity(n, W, H, ws_bytes);
  if (ecap < 0) return STP_ERR_WORKSPACE_TOO_SMALL;
  plan(n, W, H, ecap, L);
  unsigned long long c[64];
  if (cudaMemcpyAsync(c, static_cast<const unsigned char*>(ws) + L.counters, sizeof(c),
                      cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return STP_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return STP_ERR_CUDA;
  st->input = n;
  {
    unsigned long long ps[256 * 4];
    if (cudaMemcpyAsync(ps, static_cast<const unsigned char*>(ws) + L.counters + C_PSTAT * 8,
                        sizeof(ps), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return STP_ERR_CUDA;
    int64_t t[4] = {0, 0, 0, 0};
    for (int i = 0; i < 256 * 4; ++i) t[i & 3] += (int64_t)ps[i];
    st->behind = t[0];
    st->guard = t[1];
    st->degenerate = t[2];
    st->kept = t[3];
  }
  st->bin_entries = (int64_t)c[C_ENTRIES];
  st->tiles = (int64_t)c[C_TILES];
  st->nonfinite_pixels = (int64_t)c[C_NONFINITE];
  st->tie_runs = (int64_t)c[C_TIES];
  st->entry_capacity = ecap;
  st->overflow = st->bin_entries > ecap ? 1 : 0;
  if (c[C_SCHED]) {
    fprintf(stderr, "stp: K6 tile scheduler fault (%llu)\n", c[C_SCHED]);
    return STP_ERR_CUDA;
  }
  return STP_OK;
}

}  // namespace
}  // namespace stp

namespace stp {
int device_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}
}  // namespace stp

using namespace stp;

extern "C" {

int stp_abi_version(void) { return STP_ABI_VERSION; }

const char* stp_error_string(int code) {
  if (code < 0 || code > 4) return "unknown error";
  return kErrors[code];
}

int stp_validate_config(const StpConfig* cfg) { return cfg_check(cfg); }

size_t stp_workspace_bytes(int64_t n, int32_t width, int32_t height, int64_t entry_capacity) {
  StpLayout L;
  if (n < 0 || width <= 0 || height <= 0 || entry_capacity < 0) return 0;
  plan(n, width, height, entry_capacity, L);
  return L.total;
}

int stp_workspace_layout(int64_t n, int32_t width, int32_t height, size_t ws_bytes,
                         StpLayout* out) {
  if (!out || n < 0 || width <= 0 || height <= 0) return STP_ERR_CONFIG;
  const int64_t ecap = max_capacity(n, width, height, ws_bytes);
  if (ecap < 0) return STP_ERR_WORKSPACE_TOO_SMALL;
  plan(n, width, height, ecap, *out);
  return STP_OK;
}

static int check_inputs(const StpScene* scene, const StpCamera* cam, const StpConfig* cfg,
                        const StpOutputs* out) {
  if (!scene || !cam || !cfg || !out) return STP_ERR_CONFIG;
  const int rc = cfg_check(cfg);
  if (rc != STP_OK) return rc;
  if (cam->width <= 0 || cam->height <= 0 || !(cam->fx > 0) || !(cam->fy > 0))
    return STP_ERR_DATA;
  if (scene->n < 0 || (scene->n > 0 && (!scene->means || !scene->quats || !scene->scales ||
                                        !scene->opacity || !scene->sh)))
    return STP_ERR_DATA;
  if (scene->n >= (int64_t)0x7fffffff) return STP_ERR_DATA;
  const int k = scene->sh_coeffs;
  if (k != 1 && k != 4 && k != 9 && k != 16) return STP_ERR_DATA;
  if (!out->color || !out->transmittance) return STP_ERR_DATA;
  if (cfg->with_depth && !out->depth) return STP_ERR_DATA;
  if (cfg->record_cap > 0 && (!out->rec_count || !out->rec_splat || !out->rec_t ||
                              !out->rec_alpha))
    return STP_ERR_DATA;
  return STP_OK;
}

int stp_render(const StpScene* scene, const StpCamera* cam, const StpConfig* cfg, void* workspace,
               size_t workspace_bytes, const StpOutputs* out, StpStats* stats, void* stream) {
  int rc = check_inputs(scene, cam, cfg, out);
  if (rc != STP_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float ms[4] = {0, 0, 0, 0};
  const bool timed = stats && (cfg->flags & STP_FLAG_TIMINGS);
  rc = render_one(scene, nullptr, cam, cfg, workspace, workspace_bytes, out, s, nullptr, 0,
                  timed ? ms : nullptr);
  if (rc != STP_OK) return rc;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    rc = fill_stats(workspace, workspace_bytes, scene->n, cam->width, cam->height, stats, s);
    if (rc != STP_OK) return rc;
    stats->ms_project = ms[0];
    stats->ms_duplicate = ms[1];
    stats->ms_sort = ms[2];
    stats->ms_blend = ms[3];
    stats->ms_total = ms[0] + ms[1] + ms[2] + ms[3];
    if (stats->overflow) return STP_ERR_WORKSPACE_TOO_SMALL;
  }
  return STP_OK;
}

static int check_batch_inputs(const StpSplatBatch* batch, const StpCamera* cam,
                              const StpConfig* cfg, const StpOutputs* out) {
  if (!batch || !cam || !cfg || !out) return STP_ERR_CONFIG;
  const int rc = cfg_check(cfg);
  if (rc != STP_OK) return rc;
  if (cam->width <= 0 || cam->height <= 0 || !(cam->fx > 0) || !(cam->fy > 0))
    return STP_ERR_DATA;
  if (batch->n < 0 || batch->n >= (int64_t)0x7fffffff) return STP_ERR_DATA;
  if (batch->n > 0 && (!batch->mean2d || !batch->conic || !batch->color || !batch->opacity ||
                       !batch->radius || !batch->inv_cov3 || !batch->inv_cov_center))
    return STP_ERR_DATA;
  if (cfg->sort_mode == STP_MODE_GLOBALZ && batch->n > 0 &&
      (!batch->global_depth || !batch->center_dist))
    return STP_ERR_DATA;
  if (!out->color || !out->transmittance) return STP_ERR_DATA;
  if (cfg->with_depth && !out->depth) return STP_ERR_DATA;
  if (cfg->record_cap > 0 && (!out->rec_count || !out->rec_splat || !out->rec_t ||
                              !out->rec_alpha))
    return STP_ERR_DATA;
  return STP_OK;
}

int stp_render_batch(const StpSplatBatch* batch, const StpCamera* cam, const StpConfig* cfg,
                     void* workspace, size_t workspace_bytes, const StpOutputs* out,
                     StpStats* stats, void* stream) {
  int rc = check_batch_inputs(batch, cam, cfg, out);
  if (rc != STP_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float ms[4] = {0, 0, 0, 0};
  const bool timed = stats && (cfg->flags & STP_FLAG_TIMINGS);
  rc = render_one(nullptr, batch, cam, cfg, workspace, workspace_bytes, out, s, nullptr, 0,
                  timed ? ms : nullptr);
  if (rc != STP_OK) return rc;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    rc = fill_stats(workspace, workspace_bytes, batch->n, cam->width, cam->height, stats, s);
    if (rc != STP_OK) return rc;
    stats->ms_project = ms[0];
    stats->ms_duplicate = ms[1];
    stats->ms_sort = ms[2];
    stats->ms_blend = ms[3];
    stats->ms_total = ms[0] + ms[1] + ms[2] + ms[3];
    if (stats->overflow) return STP_ERR_WORKSPACE_TOO_SMALL;
  }
  return STP_OK;
}

int stp_render_views(const StpScene* scene, const StpCamera* cams, int32_t n_views,
                     const StpConfig* cfg, void* workspace, size_t workspace_bytes,
                     const StpOutputs* outs, void* stream) {
  if (n_views < 0 || (n_views > 0 && (!cams || !outs))) return STP_ERR_CONFIG;
  for (int v = 0; v < n_views; ++v) {
    int rc = check_inputs(scene, cams + v, cfg, outs + v);
    if (rc != STP_OK) return rc;
    rc = render_one(scene, nullptr, cams + v, cfg, workspace, workspace_bytes, outs + v,
                    static_cast<cudaStream_t>(stream), nullptr, 0, nullptr);
    if (rc != STP_OK) return rc;
  }
  return STP_OK;
}

int stp_render_events(const StpScene* scene, const StpCamera* cam, const StpConfig* cfg,
                      void* workspace, size_t workspace_bytes, const StpOutputs* out,
                      void* const* events, int32_t n_events, void* stream) {
  const int rc = check_inputs(scene, cam, cfg, out);
  if (rc != STP_OK) return rc;
  if (!events || (n_events != STP_STAGE_EVENTS && n_events != STP_KERNEL_EVENTS))
    return STP_ERR_CONFIG;
  cudaEvent_t ev[STP_KERNEL_EVENTS];
  for (int i = 0; i < n_events; ++i) ev[i] = static_cast<cudaEvent_t>(events[i]);
  return render_one(scene, nullptr, cam, cfg, workspace, workspace_bytes, out,
                    static_cast<cudaStream_t>(stream), ev, n_events, nullptr);
}

int stp_events_create(int32_t n, void** events) {
  for (int i = 0; i < n; ++i) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return STP_ERR_CUDA;
    events[i] = e;
  }
  return STP_OK;
}

int stp_events_destroy(int32_t n, void* const* events) {
  for (int i = 0; i < n; ++i) cudaEventDestroy(static_cast<cudaEvent_t>(events[i]));
  return STP_OK;
}

int stp_event_elapsed_ms(void* start, void* end, float* ms) {
  if (cudaEventSynchronize(static_cast<cudaEvent_t>(end)) != cudaSuccess) return STP_ERR_CUDA;
  return cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start),
                              static_cast<cudaEvent_t>(end)) == cudaSuccess
             ? STP_OK
             : STP_ERR_CUDA;
}

int stp_read_stats(const void* workspace, size_t workspace_bytes, int64_t n, int32_t width,
                   int32_t height, StpStats* stats, void* stream) {
  if (!stats) return STP_ERR_CONFIG;
  memset(stats, 0, sizeof(*stats));
  return fill_stats(workspace, workspace_bytes, n, width, height, stats,
                    static_cast<cudaStream_t>(stream));
}


static int check_grads(const StpGrads* g, int64_t n) {
  if (!g || !g->upstream || !g->pix_state) return STP_ERR_DATA;
  if (n > 0 && (!g->d_color || !g->d_opacity || !g->d_mean2d || !g->d_conic)) return STP_ERR_DATA;
  return STP_OK;
}

int stp_backward(const StpScene* scene, const StpCamera* cam, const StpConfig* cfg,
                 void* workspace, size_t workspace_bytes, const StpOutputs* out,
                 const StpGrads* grads, StpStats* stats, void* stream) {
  int rc = check_inputs(scene, cam, cfg, out);
  if (rc != STP_OK) return rc;
  if ((rc = check_grads(grads, scene->n)) != STP_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  rc = render_one(scene, nullptr, cam, cfg, workspace, workspace_bytes, out, s, nullptr, 0,
                  nullptr, grads);
  if (rc != STP_OK) return rc;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    rc = fill_stats(workspace, workspace_bytes, scene->n, cam->width, cam->height, stats, s);
    if (rc != STP_OK) return rc;
    if (stats->overflow) return STP_ERR_WORKSPACE_TOO_SMALL;
  }
  return STP_OK;
}

int stp_backward_batch(const StpSplatBatch* batch, const StpCamera* cam, const StpConfig* cfg,
                       void* workspace, size_t workspace_bytes, const StpOutputs* out,
                       const StpGrads* grads, StpStats* stats, void* stream) {
  int rc = check_batch_inputs(batch, cam, cfg, out);
  if (rc != STP_OK) return rc;
  if ((rc = check_grads(grads, batch->n)) != STP_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  rc = render_one(nullptr, batch, cam, cfg, workspace, workspace_bytes, out, s, nullptr, 0,
                  nullptr, grads);
  if (rc != STP_OK) return rc;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    rc = fill_stats(workspace, workspace_bytes, batch->n, cam->width, cam->height, stats, s);
    if (rc != STP_OK) return rc;
    if (stats->overflow) return STP_ERR_WORKSPACE_TOO_SMALL;
  }
  return STP_OK;
}

}  // extern "C"
