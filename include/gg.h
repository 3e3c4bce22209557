/* gg.h — C ABI of the B200-native batched 3D Gaussian Splatting renderer.
 *
 * The hot path of GaussGym (arXiv 2510.15352): "Gaussian splats are
 * rasterized in parallel across simulated environments ... We batch-render
 * splats across environments" (§3.2), one camera per
 * environment, "4,096 environments across 128 unique scenes" per GPU
 * (§3.3), RGB and depth from one pass (Fig. 4).
 * The per-pixel math is the 3DGS forward pass with the constants fixed in
 * SPEC.md:117-153 and SPEC.md:183; DESIGN.md §2 states every reading.
 *
 * Conventions (all functions):
 *   - Every function returns a gg_status; nothing throws or aborts across
 *     the ABI.  On failure gg_last_error(ctx) holds a one-line reason.
 *   - One context = one CUDA device = one logical thread of control; calls
 *     on a context must be externally serialised.
 *     Separate contexts (or processes) may run concurrently.
 *   - Floats are IEEE binary32, row-major, C-contiguous, no padding.
 *   - No torch types; pointers are plain host or device addresses as stated.
 */
#ifndef GG_H_
#define GG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gg_context gg_context;   /* opaque; bound to one CUDA device */

typedef enum {
  GG_OK = 0,
  GG_E_INVALID = 1,      /* bad argument (null, size <= 0, degree out of range, ...) */
  GG_E_NONFINITE = 2,    /* NaN/Inf in scene inputs; gg_last_error names the record */
  GG_E_OOM = 3,          /* device allocation failed */
  GG_E_CUDA = 4,         /* a CUDA runtime call failed */
  GG_E_BAD_SCENE = 5,    /* unknown / unloaded scene id */
  GG_E_CAPACITY = 6,     /* workspace limit exceeded */
  GG_E_UNSUPPORTED = 7   /* e.g. image too large for the tile table */
} gg_status;

/* Device-memory hook: the library allocates ALL device memory through it,
 * so the caller's allocator (e.g. the PyTorch caching allocator) stays the
 * owner.  `stream` is the cudaStream_t the memory is first used on. */
typedef struct {
  void* (*alloc)(size_t bytes, void* stream, void* user);
  void (*free)(void* ptr, void* stream, void* user);
  void* user;
} gg_allocator;

enum {
  GG_KEEP_INTERMEDIATES = 1u, /* keep opts.debug_env's integer artefacts for gg_debug_dump */
  GG_COUNTERS = 2u,           /* accumulate per-env n_eval / n_contrib totals */
  GG_ASYNC = 4u,              /* sync-free, CUDA-graph-capturable render (needs gg_reserve_async) */
  GG_TIGHT_TILES = 8u,        /* work-reduction variant (reading R35):
                                 each Gaussian's tile rect is cut to the tiles that can hold a pixel
                                 with alpha >= 1/255.  Images are bit-identical to the paper's 3-sigma
                                 rects; the tile lists (and gg_debug_dump's artefacts) are shorter. */
  GG_ELLIPSE_TILES = 16u      /* work-reduction variant (reading R37),
                                 implies GG_TIGHT_TILES: tiles of a <= 32-tile rect whose pixel centres
                                 cannot reach the alpha >= 1/255 ellipse are dropped.  Images unchanged. */
};

typedef struct {
  float near_plane;      /* metres; cull p_z <= near; default 0.01 (reading R3) */
  float far_plane;       /* metres; cull p_z > far; default 1e10 */
  float background[3];   /* rgb in [0,1] blended as C + T*bg; default 0 */
  int32_t sh_degree;     /* SH degree used at render, -1 = each scene's own (reading R18) */
  int32_t rgb_format;    /* 0 = u8 [E,H,W,3] round-half-even; 1 = f32 [E,H,W,3] */
  uint32_t flags;        /* GG_KEEP_INTERMEDIATES | GG_COUNTERS | GG_ASYNC | GG_TIGHT_TILES | GG_ELLIPSE_TILES */
  int32_t debug_env;     /* env index whose intermediates are kept (-1 = none) */
} gg_render_opts;

/* Fill `o` with the defaults above. */
void gg_default_opts(gg_render_opts* o);

/* Create a context on CUDA device `device`.  `a` may be NULL (then
 * cudaMallocAsync/cudaFreeAsync on the call's stream are used).  The
 * allocator struct is copied; its `user` pointer must outlive the context. */
gg_status gg_create(int device, const gg_allocator* a, gg_context** out);

/* Destroy the context and free every scene and workspace buffer. */
gg_status gg_destroy(gg_context* ctx);

/* Load one scene of n Gaussians (SPEC.md:28-34 SplatPrimitive; north star:
 * "gg_load_scene takes Gaussian means, scales, rotation quaternions,
 * opacities and SH colour coefficients").  Inputs are ACTIVATED values:
 *   means   [n,3] metres, world frame
 *   scales  [n,3] per-axis standard deviations, > 0 (metres)
 *   quats   [n,4] rotation (w,x,y,z), any non-zero norm (normalised here)
 *   opacities [n] in [0,1]
 *   sh      [n,(d+1)^2,3] coefficient-major SH colour (DC first; DC -> RGB
 *           via 0.2820948 f + 0.5), sh_degree d in 0..3
 * Pointers may be host or device memory (detected per pointer).  The call
 * is synchronous and COPIES the inputs (scene data is shared by all envs,
 * never copied per env); the caller may free them on return.
 * Errors (reported before anything is stored): n <= 0 ("empty ->
 * error"), d outside 0..3, null pointer -> GG_E_INVALID; NaN/Inf anywhere ->
 * GG_E_NONFINITE; scale <= 0, opacity outside [0,1], |q| = 0 -> GG_E_INVALID,
 * gg_last_error naming the first offending record index.
 * On success *out_scene_id receives the id to bind envs to. */
gg_status gg_load_scene(gg_context* ctx, int64_t n, int32_t sh_degree, const float* means,
                        const float* scales, const float* quats, const float* opacities,
                        const float* sh, int32_t* out_scene_id);

/* Release a scene's device memory; its id becomes invalid. */
gg_status gg_unload_scene(gg_context* ctx, int32_t scene_id);

/* Pre-size the workspace for renders of up to max_envs envs at width x
 * height and set the env chunk size (envs processed per pipeline pass;
 * 0 = automatic: the largest of 4096, 2048, 1024 whose workspace estimate
 * fits 80% of the device memory available when rendering; renders with host
 * outputs use at most 1024).  Optional: gg_render grows the workspace on
 * demand, and a chunk whose records or keys cannot be allocated is redone in
 * halves before GG_E_OOM is returned. */
gg_status gg_reserve(gg_context* ctx, int32_t max_envs, int32_t width, int32_t height,
                     int32_t chunk_envs);

/* Reserve the fixed workspace of the sync-free render mode (opts.flags |=
 * GG_ASYNC).  Call after loading every scene.  Renders
 * of up to max_envs envs at exactly width x height then run without any host
 * synchronisation or allocation, so they can be captured in a CUDA graph.
 * Capacities per env chunk: records = chunk * max_scene_n * max_visible_frac,
 * keys = records * keys_per_visible.  A NEGATIVE max_visible_frac = -h sizes
 * both from what earlier synchronous renders at this width x height saw
 * instead: h times the densest observed chunk's records (keys) per env times
 * the chunk, and at least h times min(chunk, 4) times the largest single env
 * seen (records capped at chunk x the largest scene); keys_per_visible is
 * then ignored (GG_E_INVALID if no such render happened).  Envs are processed in groups of 16
 * in (scene, view direction, camera position) order computed on the device
 * for up to 16384 envs (caller order beyond; outputs always go to the caller's
 * env index).  With a calibrated reservation the sort and placement run one
 * CTA per capacity block (surplus CTAs exit), otherwise bounded grids that take
 * blocks from work counters.  On overflow that chunk's frames are background
 * and gg_check_errors returns GG_E_CAPACITY.  Counters (GG_COUNTERS) are
 * supported; intermediates are not. */
gg_status gg_reserve_async(gg_context* ctx, int32_t max_envs, int32_t width, int32_t height, int32_t chunk_envs,
                           float max_visible_frac, float keys_per_visible);

/* Render one frame for each of n_envs environments (SPEC.md:154-162
 * render_batch): env e uses scene scene_ids[e] and the pinhole camera
 * (viewmats[e], intrinsics[e]).
 *   scene_ids  DEVICE int32 [E]
 *   viewmats   DEVICE f32 [E,4,4] world->camera, row-major; OpenCV axes
 *              (+x right, +y down, +z forward) (reading R2); only the top
 *              3x4 block is read
 *   intrinsics DEVICE f32 [E,4] = fx, fy, cx, cy in pixels
 *   rgb        DEVICE [E,H,W,3] u8 (rgb_format 0) or f32 (1), or NULL.  NULL selects the
 *              depth-only render (the paper's depth-only baseline): no SH
 *              colour is evaluated or blended; depth/alpha are bit-identical to the
 *              RGB+depth render.
 *   depth      DEVICE f32 [E,H,W] expected camera-z depth in metres,
 *              sum(w z)/sum(w), 0 where nothing contributes (reading R14), or NULL
 *   alpha      DEVICE f32 [E,H,W] accumulated alpha sum(w), or NULL
 * All outputs are written in stream order on `stream` (a cudaStream_t).
 * Buffers are caller-owned and must stay valid until the stream passes the
 * render.  Bit-identical results for identical inputs, independent of the
 * batch composition.  The call blocks on the stream
 * between pipeline stages of each env chunk (workspace sizing), so it
 * returns after the last chunk's kernels are enqueued.  Errors: bad args ->
 * GG_E_INVALID before any output is written; unknown scene id ->
 * GG_E_BAD_SCENE (that env is rendered as background). */
gg_status gg_render(gg_context* ctx, int32_t n_envs, const int32_t* scene_ids, const float* viewmats,
                    const float* intrinsics, int32_t width, int32_t height, const gg_render_opts* opts,
                    void* rgb, float* depth, float* alpha, void* stream);

/* Same render with HOST (ideally pinned) inputs and outputs: copies the
 * per-env inputs host->device and the frames device->host on `stream`
 * inside the call, overlapping the copy-out of chunk c with chunk c+1.
 * Synchronous: returns when the outputs are in host memory. */
gg_status gg_render_host(gg_context* ctx, int32_t n_envs, const int32_t* scene_ids,
                         const float* viewmats, const float* intrinsics, int32_t width, int32_t height,
                         const gg_render_opts* opts, void* rgb, float* depth, float* alpha,
                         void* stream);

/* Pipelined form of gg_render_host (the RL loop's double-buffered
 * observations): returns once the inputs, the render and the frame copies are
 * enqueued.  Two internal device staging slots alternate between calls, so
 * call t + 1 renders while call t's frames still stream to the host; the host
 * buffers of a call must stay valid, and must not be read, until
 * gg_host_sync returns (which waits for every outstanding frame copy).  The
 * call still blocks on the render stream between the pipeline stages of each
 * env chunk (workspace sizing), as gg_render does.  GG_ASYNC is not accepted
 * here (GG_E_UNSUPPORTED). */
gg_status gg_render_host_async(gg_context* ctx, int32_t n_envs, const int32_t* scene_ids,
                               const float* viewmats, const float* intrinsics, int32_t width, int32_t height,
                               const gg_render_opts* opts, void* rgb, float* depth, float* alpha,
                               void* stream);
gg_status gg_host_sync(gg_context* ctx);

/* Motion blur (§3.3 "rendering a small set of frames offset
 * along the camera's velocity direction and alpha-blending them into a
 * single image"; SPEC.md:221-229 render_with_motion_blur).  Readings
 * (R32-R34): sample times t_i = shutter*((i+0.5)/K - 0.5),
 * i = 0..K-1; sample pose i rotates the camera about its centre by the
 * axis-angle vector ang_vel*t_i (world frame) and moves the centre by
 * lin_vel*t_i (world frame, m/s); the K renders are averaged in linear f32
 * colour before quantisation as m = x_0 + (sum_{i>=1} (x_i - x_0)) / K (so K=1
 * and zero velocity reproduce the static render bit-exactly); alpha is
 * averaged the same way; depth is taken from sample floor(K/2).
 *   lin_vel, ang_vel  DEVICE f32 [E,3]; shutter >= 0 seconds; K in 1..64
 * Other arguments and outputs as gg_render. */
gg_status gg_render_blur(gg_context* ctx, int32_t n_envs, const int32_t* scene_ids, const float* viewmats,
                         const float* intrinsics, const float* lin_vel, const float* ang_vel, float shutter,
                         int32_t K, int32_t width, int32_t height, const gg_render_opts* opts, void* rgb,
                         float* depth, float* alpha, void* stream);

/* The K sample view matrices gg_render_blur renders: DEVICE f32 [E,K,4,4]
 * (bottom row 0,0,0,1).  Exposed for tests. */
gg_status gg_blur_poses(gg_context* ctx, int32_t n_envs, const float* viewmats, const float* lin_vel,
                        const float* ang_vel, float shutter, int32_t K, float* out_viewmats, void* stream);

/* Deterministic 64-bit digest per env of the outputs just rendered
 * (rgb bytes and depth bits), written to DEVICE uint64 [E] on stream.
 * Used for cross-GPU / batch-composition determinism checks. */
gg_status gg_checksum(gg_context* ctx, int32_t n_envs, int32_t width, int32_t height,
                      const void* rgb, int32_t rgb_format, const float* depth, uint64_t* out,
                      void* stream);

/* Rendered frames -> DinoV2 input ("DinoV2
 * embeddings extracted from the raw RGB frame"; reading R36):
 *   rgb   DEVICE u8 [E,H,W,3] (gg_render's rgb_format 0 output)
 *   out   DEVICE bf16 [E,3,S,S]: bilinear resize (half-pixel centres, no
 *         antialiasing) of the whole frame to S x S, /255, ImageNet mean/std,
 *         round-to-nearest-even, channel-planar.  Caller-owned.
 * Enqueued on `stream`; GG_E_INVALID for null pointers or sizes <= 0. */
gg_status gg_dino_input(gg_context* ctx, int32_t n_envs, int32_t width, int32_t height, const uint8_t* rgb,
                        int32_t size, void* out_bf16, void* stream);

/* 3DGS binary PLY scenes (SPEC.md:51-59 load_splat_ply).
 * gg_read_ply parses `path` into ACTIVATED host arrays (scale = exp,
 * opacity = sigmoid, quaternion = rot_0..3 as (w,x,y,z), SH reordered from
 * the file's channel-major f_rest to [n,(d+1)^2,3]).  Call once with null
 * array pointers to get n and the SH degree, then with caller-allocated
 * host buffers of those sizes.  Errors: missing property (named), NaN/Inf
 * (record index), empty or truncated file -> GG_E_INVALID with the reason in
 * gg_ply_error().  No context or GPU needed.  gg_load_ply = gg_read_ply +
 * gg_load_scene. */
gg_status gg_read_ply(const char* path, int64_t* n, int32_t* sh_degree, float* means, float* scales,
                      float* quats, float* opacities, float* sh);
gg_status gg_load_ply(gg_context* ctx, const char* path, int32_t* out_scene_id);
const char* gg_ply_error(void);

/* Synchronise `stream` and return any sticky device-side error. */
gg_status gg_check_errors(gg_context* ctx, void* stream);

/* Intermediates of opts.debug_env from the last render with
 * GG_KEEP_INTERMEDIATES (test only).  Copies up to `capacity` elements into
 * host_dst and stores the full length in *out_len.  Kinds:
 *   GG_DUMP_TILE_COUNTS   int32 [N]   tiles per Gaussian (0 if culled)
 *   GG_DUMP_SORTED_TILE   int32 [K]   tile of each sorted entry
 *   GG_DUMP_SORTED_ZBITS  uint32 [K]  f32 bits of the view depth
 *   GG_DUMP_SORTED_GIDS   int32 [K]   Gaussian index
 *   GG_DUMP_RANGES        int32 [T,2] [start,end) per tile
 *   GG_DUMP_COUNTERS      int64 [4]   sum n_eval, sum n_contrib, V, K of that env
 *   GG_DUMP_N_EVAL        int32 [H*W] per-pixel visited count (needs GG_COUNTERS)
 *   GG_DUMP_PROJ          float [N,16] vis,u,v,A,B,C,z,r,x0,x1,y0,y1,r,g,b,o   */
enum {
  GG_DUMP_TILE_COUNTS = 0, GG_DUMP_SORTED_TILE = 1, GG_DUMP_SORTED_ZBITS = 2,
  GG_DUMP_SORTED_GIDS = 3, GG_DUMP_RANGES = 4, GG_DUMP_COUNTERS = 5, GG_DUMP_N_EVAL = 6,
  GG_DUMP_PROJ = 7
};
gg_status gg_debug_dump(gg_context* ctx, int32_t kind, void* host_dst, int64_t capacity,
                        int64_t* out_len);

/* Per-env counters of the last render with GG_COUNTERS, copied to host
 * int64 [E,4]: n_eval sum, n_contrib sum, visible records V, keys K. */
gg_status gg_get_counters(gg_context* ctx, int32_t n_envs, int64_t* host_dst);

/* Number of kernels this context has launched since creation. */
int64_t gg_launch_count(const gg_context* ctx);

/* Envs per pipeline pass (chunk) of the last render (0 before any). */
int32_t gg_chunk_envs(const gg_context* ctx);

/* Per-stage device time (ms) of the last render, measured with CUDA events on
 * the render stream when `enable` was set by gg_set_timing (events are
 * resolved lazily: the first query after a render synchronises with it).
 * gg_get_stage_ms: 3 stages = project (cull + project), sort (depth passes +
 * placement), raster.  gg_get_stage_times: the first n (1..5) of the finer
 * stages cull (K1a + K2), project (K1b), depth passes (K3/K4 depth),
 * placement (K4/K5 tile pass + ranges), raster (K6).  In the host-synchronising
 * sync mode the project stage also spans the host's per-chunk readback. */
gg_status gg_set_timing(gg_context* ctx, int32_t enable);
gg_status gg_get_stage_ms(gg_context* ctx, float* out3);
gg_status gg_get_stage_times(gg_context* ctx, float* out, int32_t n);

const char* gg_last_error(const gg_context* ctx);
const char* gg_status_string(gg_status s);

#ifdef __cplusplus
}
#endif
#endif /* GG_H_ */
