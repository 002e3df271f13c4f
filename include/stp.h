/*
 * stp.h — C ABI of the B200 hierarchical Gaussian-splatting forward renderer.
 *
 * Drop-in boundary for the reference's render path
 *   render(scene, cam, Hierarchical(), cfg) -> FrameOutput
 *   (/root/reference/pkg/src/splatsort/rasterizer.py:595-698)
 * with the per-stage seams
 *   project_scene   gaussian_math.py:323-434     (kernel K1)
 *   bin_and_sort    rasterizer.py:279-377         (K2 scan, K3 duplicate, K4 sort, K5 ranges)
 *   render_tile     hierarchy.py:27-219           (K6)
 *
 * Plain pointers and sizes only (no torch types).  All array pointers in
 * StpScene / StpOutputs are DEVICE pointers; StpCamera / StpConfig / StpStats
 * are host structs passed by pointer.  Every call is asynchronous on the given
 * cudaStream_t (passed as void*), re-entrant per (workspace, stream) and
 * deterministic.  No exceptions cross the ABI: every entry point returns a
 * status code (errors.py:4-13 mapping below).
 */
#ifndef STP_H_
#define STP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STP_ABI_VERSION 3

/* Status codes.  CONFIG -> ConfigError (rasterizer.py:93-117, 196-203),
 * DATA -> DataError (rasterizer.py:770-771), WORKSPACE_TOO_SMALL -> the host
 * grows the workspace to the frame's entry count and retries once.  The entry
 * count E of a frame is only known on the device after K3: synchronous calls
 * (stats != NULL) return WORKSPACE_TOO_SMALL with StpStats.bin_entries = E;
 * asynchronous calls report it through StpOutputs.status (below), which the
 * caller reads after synchronising the stream. */
enum {
  STP_OK = 0,
  STP_ERR_CONFIG = 1,
  STP_ERR_DATA = 2,
  STP_ERR_WORKSPACE_TOO_SMALL = 3,
  STP_ERR_CUDA = 4
};

/* Scene tensors, drop-in layout of Gaussian3D stacked as in
 * gaussian_math.py:353-357 (float32, C-contiguous, device memory). */
typedef struct {
  const float* means;     /* [n,3] world-space centres                      */
  const float* quats;     /* [n,4] quaternion w,x,y,z (re-normalised inside) */
  const float* scales;    /* [n,3] per-axis standard deviations             */
  const float* opacity;   /* [n]   linear opacity                           */
  const float* sh;        /* [n,sh_coeffs,3] SH coefficients [k][rgb]       */
  int64_t n;
  int32_t sh_coeffs;      /* 1, 4, 9 or 16 (degree 0..3)                    */
  int32_t reserved;
} StpScene;

/* An already-projected SplatBatch (gaussian_math.py:260-307), the other
 * input render() accepts (rasterizer.py:616-618): float64 device arrays, the
 * batch index is the rank.  Opacity and colour are rounded to float32 (they
 * only scale alpha and the blended colour; every geometric decision uses the
 * float64 fields). */
typedef struct {
  const double* mean2d;          /* [n,2]                                      */
  const double* conic;           /* [n,3] a, b, c                              */
  const double* color;           /* [n,3]                                      */
  const double* opacity;         /* [n]                                        */
  const double* radius;          /* [n]                                        */
  const double* inv_cov3;        /* [n,6] packed m00, m11, m22, m01, m02, m12  */
  const double* inv_cov_center;  /* [n,3]                                      */
  int64_t n;
  const double* global_depth;    /* [n] view z (GlobalZ keys) or NULL           */
  const double* center_dist;     /* [n] |mean - origin| (GlobalZ depth) or NULL */
} StpSplatBatch;

/* Pinhole camera (scene_io.py:84-129): world->view rotation, row-major. */
typedef struct {
  double R[9];
  double pos[3];
  double fx, fy, cx, cy;
  int32_t width, height;
} StpCamera;

/* RenderConfig (rasterizer.py:170-208) + Hierarchical (rasterizer.py:70-87). */
typedef struct {
  double eps;               /* opacity_eps, 1/255                          */
  double termination;       /* 1e-4                                        */
  double alpha_cap;         /* 0.99                                        */
  double bg[3];             /* background                                  */
  double near_plane;        /* 0.2                                         */
  double guard;             /* 1.3                                         */
  double dilation;          /* 0.3                                         */
  double inv_scale_clamp;   /* 1e3                                         */
  int32_t tile_size;        /* must be 16                                  */
  int32_t q_tail, q_mid, q_head;   /* queue sizes (64/8/4)                 */
  int32_t b_load, b_mid, b_head;   /* batches; must be 32/16/4             */
  int32_t mid_depth_at_center;
  int32_t with_depth;
  int32_t exact_culling;    /* exact 16x16 tile culling (default 1)        */
  int32_t record_cap;       /* per-pixel blend-record capacity, 0 = off    */
  int32_t flags;            /* STP_FLAG_*                                  */
  int32_t sort_mode;        /* STP_MODE_* (rasterizer.py:89 SortMode)      */
  int32_t tile_begin;       /* K6 renders tiles [tile_begin, tile_end) only */
  int32_t tile_end;         /*   (row-major tile ids; 0, 0 = every tile):   */
                            /*   a band of a view split across GPUs; K1-K5 */
                            /*   run for the whole view, only the band's   */
                            /*   pixels are written                        */
} StpConfig;

/* Sort modes.  HIERARCHICAL: per-tile t_opt keys + the 3-level resort
 * (hierarchy.py); GLOBALZ: one view-space z key per splat and the bin's
 * order for every pixel (rasterizer.py:472-485, the 3DGS baseline);
 * FULL: the exact per-pixel order (rasterizer.py:488-501); WINDOW: a
 * per-pixel resorting window of q_head entries over the per-tile-key stream
 * (rasterizer.py:504-588, Window.size -> q_head, 1..STP_WINDOW_MAX: a
 * register window up to 16, a per-pixel shared-memory heap above).  Queue
 * fields other than q_head (WINDOW) are ignored outside HIERARCHICAL. */
#define STP_MODE_HIERARCHICAL 0
#define STP_MODE_GLOBALZ 1
#define STP_MODE_FULL 2
#define STP_MODE_WINDOW 3
#define STP_WINDOW_MAX 512

#define STP_FLAG_TIMINGS 1  /* record per-stage CUDA-event timings (syncs) */

/* Output buffers (device).  Colour is HWC float32 composited over the
 * background (rasterizer.py:680); depth is the unnormalised expected depth
 * sum(w * t) (hierarchy.py:88).  Records, when record_cap > 0, hold the first
 * record_cap blended contributions of each pixel in blend order
 * (hierarchy.py:89-90); rec_splat is the Gaussian (source) index. */
typedef struct {
  float* color;          /* [H,W,3]                        */
  float* transmittance;  /* [H,W]                          */
  float* depth;          /* [H,W] or NULL                  */
  int32_t* rec_count;    /* [H,W] or NULL                  */
  int32_t* rec_splat;    /* [H,W,record_cap]               */
  float* rec_t;          /* [H,W,record_cap]               */
  float* rec_alpha;      /* [H,W,record_cap]               */
  uint8_t* state;        /* [n] per-Gaussian cull state or NULL:
                            0 kept, 1 behind, 2 guard, 3 degenerate      */
  float* sort_error;     /* [H,W] per-pixel sort error delta or NULL: the sum
                            of positive depth inversions of consecutive blended
                            contributions (metrics.py:46-73)             */
  int64_t* status;       /* [2] frame status word or NULL, written on the
                            device by K5 (and K6): status[0] = STP_OK, or
                            STP_ERR_WORKSPACE_TOO_SMALL when the frame's
                            entries exceeded the workspace capacity (the
                            frame is then truncated and must be re-rendered
                            with a larger workspace), or STP_ERR_CUDA on an
                            internal scheduler fault; status[1] = the frame's
                            entry count E.  The asynchronous paths' error
                            report (stp_render(stats = NULL),
                            stp_render_events, one word per view in
                            stp_render_views).                              */
  /* float64 outputs (the reference's FrameOutput precision, rasterizer.py:
   * 246-255), all optional.  With color64 set, K6 also accumulates each
   * pixel's colour and depth in float64 and composites the background in
   * float64 (the float32 buffers above are still written); rec_t64 /
   * rec_alpha64 receive the blend records' t and alpha in float64. */
  double* color64;          /* [H,W,3] or NULL                              */
  double* transmittance64;  /* [H,W]   (with color64)                       */
  double* depth64;          /* [H,W]   or NULL (with color64)               */
  double* rec_t64;          /* [H,W,record_cap] or NULL                     */
  double* rec_alpha64;      /* [H,W,record_cap] or NULL                     */
  double* splat_color64;    /* [n,3] scratch or NULL (with color64, Gaussian
                               input): the SH colour in float64
                               (gaussian_math.py:415-419), blended instead of
                               the float32 record colour.  A SplatBatch input
                               blends its own float64 colour.               */
} StpOutputs;

/* stats dict of rasterizer.py:683-690 (+ projection stats
 * gaussian_math.py:344) and per-stage device timings in milliseconds. */
typedef struct {
  int64_t input, behind, guard, degenerate, kept;
  int64_t bin_entries;      /* exact-culled (tile, splat) entries          */
  int64_t tiles;            /* non-empty tiles                             */
  int64_t nonfinite_pixels;
  int64_t tie_runs;         /* equal fp32 keys re-ordered by fp64 depth    */
  int64_t entry_capacity;   /* workspace capacity used for this frame      */
  float ms_project, ms_duplicate, ms_sort, ms_blend, ms_total;
  int32_t overflow;         /* 1 if bin_entries > entry_capacity           */
} StpStats;

/* Byte offsets of the workspace regions (debug / parity dumps). */
typedef struct {
  size_t recs, camera, masks, state, counts, offsets, keys0, keys1, vals, ranges,
      counters, hist, lookback, scan_scratch,
      rowlist, /* ids of kept Gaussians whose coarse rect exceeds 64 tiles */
      aux,     /* [n] (view z, |mean - origin|) float64 pairs (GlobalZ)     */
      total;
  int64_t entry_capacity;
  int32_t n_tiles, grid_w, grid_h, sort_passes, sort_bits, partitions;
  int32_t splat_record_bytes;
  int32_t final_buffer;     /* sorted entry words in keys0 (0) or keys1 (1)     */
  int32_t depth_bits;       /* entry word = (tile << depth_bits |               */
  int32_t id_bits;          /*   depth key >> (32 - depth_bits)) << id_bits | id */
} StpLayout;

int stp_abi_version(void);
const char* stp_error_string(int code);

/* STP_OK or STP_ERR_CONFIG (same rules as validate_mode / RenderConfig). */
int stp_validate_config(const StpConfig* cfg);

/* Workspace needed for n Gaussians, a width x height frame and up to
 * entry_capacity (tile, splat) entries. */
size_t stp_workspace_bytes(int64_t n, int32_t width, int32_t height, int64_t entry_capacity);

/* Region offsets for a workspace of ws_bytes (entry capacity is derived). */
int stp_workspace_layout(int64_t n, int32_t width, int32_t height, size_t ws_bytes,
                         StpLayout* out);

/* Render one view.  Asynchronous unless `stats` is non-NULL (then the stream
 * is synchronised and the stats filled; an entry overflow returns
 * STP_ERR_WORKSPACE_TOO_SMALL with stats->bin_entries set). */
int stp_render(const StpScene* scene, const StpCamera* cam, const StpConfig* cfg,
               void* workspace, size_t workspace_bytes, const StpOutputs* out,
               StpStats* stats, void* stream);

/* Render an already-projected SplatBatch (projection skipped, as in
 * rasterizer.py:616-618); otherwise identical to stp_render. */
int stp_render_batch(const StpSplatBatch* batch, const StpCamera* cam, const StpConfig* cfg,
                     void* workspace, size_t workspace_bytes, const StpOutputs* out,
                     StpStats* stats, void* stream);

/* Render n_views cameras back to back on one stream (one workspace, outputs
 * per view); never synchronises.  Entry overflow of view v is reported in
 * outs[v].status (set it to detect overflow: the shared workspace is
 * overwritten by the next view, so it cannot be recovered afterwards). */
int stp_render_views(const StpScene* scene, const StpCamera* cams, int32_t n_views,
                     const StpConfig* cfg, void* workspace, size_t workspace_bytes,
                     const StpOutputs* outs, void* stream);

/* Render one view recording caller-created CUDA events (cudaEvent_t as
 * void*) at kernel boundaries; asynchronous.  n_events = 5: the stage
 * boundaries [K0+K1 | K2+K3 | K4+K5 | K6] (rasterizer.py:299-376 timing keys
 * project / duplicate / sort / blend); n_events = 8: every kernel
 * [K0 init | K1 preprocess (+ row count) | K2 scan | K3 duplicate (+ row
 * duplicate) | K4 sort | K5 ranges | K6 render].  The last interval brackets
 * the render kernel K6 alone. */
#define STP_STAGE_EVENTS 5
#define STP_KERNEL_EVENTS 8
int stp_render_events(const StpScene* scene, const StpCamera* cam, const StpConfig* cfg,
                      void* workspace, size_t workspace_bytes, const StpOutputs* out,
                      void* const* events, int32_t n_events, void* stream);

/* Backward pass (gradients.py:103-162): gradients of the loss w.r.t. the
 * projected splat attributes, given dL/d(colour) of the frame.  The frame is
 * rendered again into `out` and K6 is replayed twice over the same bins (the
 * blend order is recomputed, no records are stored): first for each pixel's
 * float64 colour sum and final T (pix_state), then with every blended
 * contribution's gradients added (float64 atomics) by Gaussian id -- the
 * SplatBatch index for stp_backward_batch.  d_background = sum upstream * T
 * is left to the caller (pix_state[..., 3] holds T).  Any sort mode. */
typedef struct {
  const double* upstream;  /* [H,W,3] dL/d colour                          */
  double* pix_state;       /* [H,W,4] scratch: colour sum (3), final T     */
  double* d_color;         /* [n,3]   (zeroed by the call)                 */
  double* d_opacity;       /* [n]                                          */
  double* d_mean2d;        /* [n,2]                                        */
  double* d_conic;         /* [n,3]   (a, b, c) of the conic               */
} StpGrads;

int stp_backward(const StpScene* scene, const StpCamera* cam, const StpConfig* cfg,
                 void* workspace, size_t workspace_bytes, const StpOutputs* out,
                 const StpGrads* grads, StpStats* stats, void* stream);
int stp_backward_batch(const StpSplatBatch* batch, const StpCamera* cam, const StpConfig* cfg,
                       void* workspace, size_t workspace_bytes, const StpOutputs* out,
                       const StpGrads* grads, StpStats* stats, void* stream);

/* Thin cudart helpers so hosts without a CUDA binding can time stages. */
int stp_events_create(int32_t n, void** events);
int stp_events_destroy(int32_t n, void* const* events);
int stp_event_elapsed_ms(void* start, void* end, float* ms);

/* Read the stats of the last frame rendered into `workspace` (synchronises
 * the stream). */
int stp_read_stats(const void* workspace, size_t workspace_bytes, int64_t n, int32_t width,
                   int32_t height, StpStats* stats, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STP_H_ */
