// api.cu — the C ABI of include/gg.h: context, scene store, workspace and
// the per-chunk render pipeline (K1a -> K2 -> K1b -> K3-5 -> K6).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gg.h"
#include "gg_internal.cuh"

namespace gg {
void launch_validate(int64_t n, int K, const float* means, const float* scales, const float* quats,
                     const float* opac, const float* sh, ValidateOut* out, cudaStream_t s);
void launch_pack(int64_t n, int K, int sh_stride, const float* means, const float* scales,
                 const float* quats, const float* opac, const float* sh, const uint32_t* perm, float4* pos_op,
                 float4* cov_a, float4* cov_b, float2* aux, float* qmax, float* sh_out, uint32_t* gid_out,
                 cudaStream_t s);
int launch_spatial_order(int64_t n, const float* means, uint32_t* box, uint32_t* tmp, uint32_t* hist,
                         uint32_t* perm, cudaStream_t s);
void launch_block_bounds(int n, const float4* pos_op, const float2* aux, float4* bbox, cudaStream_t s);
bool launch_env_order(int E, const int32_t* scene_ids, const float* viewmats, int nscenes, const DevScene* scenes,
                      int32_t* perm, cudaStream_t s);
void launch_setup_envs(int E, const int32_t* perm, const int32_t* scene_ids, const float* viewmats,
                       const float* intr, const DevScene* scenes, int nscenes, int W, int H, int sh_degree,
                       EnvConst* out, uint32_t* err, cudaStream_t s);
void launch_cull_count(int e0, int ngroups, int nblk, int bpc, const EnvGroup* groups, const EnvConst* envs,
                       const DevScene* scenes, const RenderParams& rp, const ChunkWS& ws, cudaStream_t s);
void launch_scan_blocks(int ec, int nblk, uint32_t* data, uint32_t* totals, cudaStream_t s);
void launch_project(int e0, int ngroups, int nblk, int bpc, int max_degree, const EnvGroup* groups,
                    const EnvConst* envs, const DevScene* scenes, const RenderParams& rp, const ChunkWS& ws,
                    cudaStream_t s);
cudaError_t project_init();
cudaError_t sort_bin_init();
uint32_t sort_blocks(uint32_t V);
int sort_block_size();
size_t sort_ghist_words();
int depth_passes(uint32_t span);
int launch_sort_bin(int ec, uint32_t nb, const uint32_t* blk_base, uint32_t* blk_env, int passes,
                    const RenderParams& rp,
                    const ChunkWS& ws, uint32_t* ghist, uint32_t* thist, cudaStream_t s, bool nb_is_capacity,
                    uint32_t* qctr, cudaEvent_t after_depth);
void launch_raster(int e0, int ec, const EnvConst* envs, const RenderParams& rp, const ChunkWS& ws, void* rgb,
                   float* depth, float* alpha, bool counters, unsigned long long* env_counts, int32_t* dbg_neval,
                   int dbg_eloc, cudaStream_t s);
void launch_blur_poses(int E, int K, int Kc, const float* viewmats, const float* lin, const float* ang,
                       float shutter, float* out, cudaStream_t s);
void launch_blur_expand(int ec, int K, const int32_t* ids, const float* intr, int32_t* ids_k, float* intr_k,
                        cudaStream_t s);
void launch_tables_v(int ec, const uint32_t* vcnt, uint64_t* rbase, uint64_t vcap, uint32_t* ok, uint32_t* err,
                     cudaStream_t s);
void launch_tables_k(int ec, const uint32_t* vcnt, const unsigned long long* kcnt, uint64_t* kbase, uint32_t* blkbase,
                     int sort_blk, uint64_t kcap, uint64_t nbcap, uint32_t* ok, uint32_t* err, cudaStream_t s);
void launch_checksum(int E, int W, int H, const uint8_t* rgb8, const float* rgbf, const float* depth,
                     unsigned long long* out, cudaStream_t s);
void launch_dino_input(int E, int W, int H, int S, const uint8_t* rgb, void* out, cudaStream_t s);
int launch_copy_words(void* dst, const void* src, size_t bytes, cudaStream_t s);
void launch_debug_records(uint32_t V, uint64_t rb, const ChunkWS& ws, int32_t* tile_counts, float* proj,
                          cudaStream_t s);
void launch_debug_sorted(int ntiles, const uint2* ranges, uint64_t kb, uint64_t rb, const ChunkWS& ws,
                         int32_t* s_tile, uint32_t* s_z, int32_t* s_gid, cudaStream_t s);
}  // namespace gg

using namespace gg;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

// Per-call workspace.  The sync path and the sync-free (GG_ASYNC) path own
// separate sets: a CUDA graph captured over a GG_ASYNC render holds the
// addresses of `aw`, which only gg_reserve_async (re)allocates, so a later
// sync render that grows its own buffers never frees memory a graph uses.
struct Work {
  DevBuf envc, flags, blkcnt, vcnt, kcnt, rbase, kbase;
  DevBuf rec0, rec1, rec2, rect, zkey, gid, dk0, dv0, dk1, rmask, dconic;
  DevBuf sorted, ranges, counters, perm, groups, blkbase, blkenv, ghist, thist, qctr, okflag;
  DevBuf* all() { return &envc; }
  static constexpr int count = 29;
};
static_assert(sizeof(Work) == Work::count * sizeof(DevBuf), "Work::count");

struct SceneSlot {
  DevScene d{};
  DevBuf pos_op, cov_a, cov_b, aux, qmax, sh, gid, bbox;
  bool live = false;
  void free_all(gg_context* ctx, cudaStream_t s);
};

constexpr int DEFAULT_CHUNK = 0;   // 0 = auto: the largest of 4096 / 2048 / 1024 envs the free memory allows
// timed stages: cull+scan, project, depth passes, placement (+ranges), raster
constexpr int NSTAGE = 5;
constexpr int SCENE_TABLE_MIN = 4096;   // scene-table slots allocated up front

}  // namespace

struct gg_context {
  int device = 0;
  gg_allocator alloc{};
  bool has_alloc = false;
  cudaStream_t own = nullptr;   // load-time work + copy-out stream
  std::string err;
  int64_t launches = 0;
  std::vector<SceneSlot> scenes;
  DevBuf scene_table;
  int scene_table_cap = 0;
  int chunk = DEFAULT_CHUNK;
  int last_chunk = 0;   // envs per pass of the last render
  int ac_E = -1, ac_chunk = 0;   // auto_chunk cache
  double ac_bytes = 0.0;
  const void* ac_set = nullptr;
  // observed by synchronous renders (calibrates gg_reserve_async): the
  // densest chunk's records and keys per env, the largest single env, and
  // the image size they were seen at
  double cal_vmean = 0.0, cal_kmean = 0.0;
  uint64_t cal_vmax = 0, cal_kmax = 0;
  int cal_W = 0, cal_H = 0;
  // workspace: sync path (sw) and sync-free path (aw), see Work
  Work sw, aw;
  const DevBuf* last_counters = nullptr;   // counters buffer of the last render
  DevBuf errflag, valid_out;
  DevBuf dbg_tc, dbg_proj, dbg_stile, dbg_sz, dbg_sgid, dbg_neval;
  DevBuf h_in[2];   // device staging of gg_render_host(_async) (ids | viewmats | intr | outputs), ping-pong
  cudaEvent_t h_done[2] = {nullptr, nullptr};   // end of the frame copies of the call that last used slot i
  bool h_pending[2] = {false, false};
  int h_slot = 0;
  DevBuf blur_vm, blur_ids, blur_intr;   // gg_render_blur sample cameras
  // pinned host mirrors
  uint32_t* h_vcnt = nullptr;
  uint64_t* h_kcnt = nullptr;
  uint64_t* h_rbase = nullptr;
  uint64_t* h_kbase = nullptr;
  uint32_t* h_err = nullptr;
  int32_t* h_ids = nullptr;
  float* h_vm = nullptr;        // view matrices (env ordering key)
  int32_t* h_perm = nullptr;
  EnvGroup* h_groups = nullptr;
  uint32_t* h_blkbase = nullptr;
  int h_cap = 0;
  // debug snapshot (host)
  std::vector<int32_t> d_tc, d_stile, d_sgid, d_ranges, d_neval;
  std::vector<uint32_t> d_sz;
  std::vector<float> d_proj;
  int64_t d_counters[4] = {0, 0, 0, 0};
  // timing
  bool timing = false;
  float stage_ms[NSTAGE] = {0, 0, 0, 0, 0};
  std::vector<cudaEvent_t> tev;   // per-chunk stage events [chunk][NSTAGE + 1], resolved lazily
  int t_nchunks = 0;              // chunks of the last timed render not yet resolved
  bool t_append = false;          // gg_render_blur: its render_impl calls add to one timing record
  cudaEvent_t ev_copy = nullptr;
  int last_E = 0;
  // sync-free mode (gg_reserve_async)
  bool async_ready = false;
  int a_max_envs = 0, a_W = 0, a_H = 0, a_chunk = 0, a_nblk = 0, a_maxdeg = 0;
  uint64_t a_vcap = 0, a_kcap = 0, a_nbcap = 0;
  bool a_loop = true;   // async sort/placement: bounded-grid work-counter kernels (else capacity-sized grids)
  DevBuf okflag;
};

namespace {

gg_status fail(gg_context* c, gg_status s, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return s;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(ctx, GG_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

void* dev_alloc(gg_context* ctx, size_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  if (ctx->has_alloc) return ctx->alloc.alloc(bytes, (void*)s, ctx->alloc.user);
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dev_free(gg_context* ctx, DevBuf& b, cudaStream_t s) {
  if (b.p) {
    if (ctx->has_alloc)
      ctx->alloc.free(b.p, (void*)s, ctx->alloc.user);
    else
      cudaFreeAsync(b.p, s);
  }
  b.p = nullptr;
  b.bytes = 0;
}

void SceneSlot::free_all(gg_context* ctx, cudaStream_t s) {
  for (DevBuf* b : {&pos_op, &cov_a, &cov_b, &aux, &qmax, &sh, &gid, &bbox}) dev_free(ctx, *b, s);
}

// grow-only buffer
bool ensure(gg_context* ctx, DevBuf& b, size_t bytes, cudaStream_t s) {
  if (b.bytes >= bytes && b.p) return true;
  if (b.p) cudaDeviceSynchronize();   // growth is rare; never free under in-flight work
  dev_free(ctx, b, s);
  const size_t nb = std::max<size_t>(bytes + bytes / 8, 256);
  b.p = dev_alloc(ctx, nb, s);
  if (!b.p) return false;
  b.bytes = nb;
  return true;
}

// Pinned host mirrors of the per-chunk tables.  All-or-nothing: the new set
// is allocated into temporaries and swapped in only when every allocation
// succeeded, so a failure leaves the old (valid) set and h_cap untouched.
bool ensure_host(gg_context* ctx, int n) {
  if (ctx->h_cap >= n) return true;
  cudaDeviceSynchronize();   // in-flight copy kernels may still read/write the old mirrors
  const int cap = std::max(n, 1024);
  void* p[9] = {};
  const size_t sz[9] = {(size_t)(cap + 1) * 4, (size_t)cap * 4, (size_t)cap * 4, (size_t)cap * sizeof(EnvGroup),
                        (size_t)cap * 4, (size_t)cap * 8, (size_t)cap * 8, (size_t)cap * 8, (size_t)cap * 64};
  for (int i = 0; i < 9; ++i) {
    if (cudaMallocHost(&p[i], sz[i]) != cudaSuccess) {
      cudaGetLastError();
      for (int j = 0; j < i; ++j) cudaFreeHost(p[j]);
      return false;
    }
  }
  void** cur[9] = {(void**)&ctx->h_blkbase, (void**)&ctx->h_ids, (void**)&ctx->h_perm, (void**)&ctx->h_groups,
                   (void**)&ctx->h_vcnt, (void**)&ctx->h_kcnt, (void**)&ctx->h_rbase, (void**)&ctx->h_kbase,
                   (void**)&ctx->h_vm};
  for (int i = 0; i < 9; ++i) {
    if (*cur[i]) cudaFreeHost(*cur[i]);
    *cur[i] = p[i];
  }
  ctx->h_cap = cap;
  return true;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int max_scene_n(const gg_context* ctx) {
  int m = 0;
  for (const auto& s : ctx->scenes)
    if (s.live) m = std::max(m, s.d.n);
  return m;
}

template <typename T>
T* P(const DevBuf& b) {
  return reinterpret_cast<T*>(b.p);
}

}  // namespace

extern "C" {

void gg_default_opts(gg_render_opts* o) {
  if (!o) return;
  o->near_plane = 0.01f;
  o->far_plane = 1e10f;
  o->background[0] = o->background[1] = o->background[2] = 0.f;
  o->sh_degree = -1;
  o->rgb_format = 0;
  o->flags = 0;
  o->debug_env = -1;
}

const char* gg_status_string(gg_status s) {
  switch (s) {
    case GG_OK: return "GG_OK";
    case GG_E_INVALID: return "GG_E_INVALID";
    case GG_E_NONFINITE: return "GG_E_NONFINITE";
    case GG_E_OOM: return "GG_E_OOM";
    case GG_E_CUDA: return "GG_E_CUDA";
    case GG_E_BAD_SCENE: return "GG_E_BAD_SCENE";
    case GG_E_CAPACITY: return "GG_E_CAPACITY";
    case GG_E_UNSUPPORTED: return "GG_E_UNSUPPORTED";
  }
  return "GG_E_?";
}

const char* gg_last_error(const gg_context* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t gg_launch_count(const gg_context* ctx) { return ctx ? ctx->launches : 0; }

int32_t gg_chunk_envs(const gg_context* ctx) { return ctx ? ctx->last_chunk : 0; }

gg_status gg_create(int device, const gg_allocator* a, gg_context** out) {
  gg_context* ctx = nullptr;
  if (!out) return GG_E_INVALID;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return GG_E_CUDA;
  }
  ctx = new gg_context();
  ctx->device = device;
  if (a && a->alloc && a->free) {
    ctx->alloc = *a;
    ctx->has_alloc = true;
  }
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking));
  CK(sort_bin_init());
  CK(project_init());
  CK(cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming));
  CK(cudaMallocHost(&ctx->h_err, 4));
  if (!ensure_host(ctx, 1024)) return fail(ctx, GG_E_OOM, "pinned host alloc failed");
  if (!ensure(ctx, ctx->errflag, 4, ctx->own)) return fail(ctx, GG_E_OOM, "alloc");
  CK(cudaMemsetAsync(ctx->errflag.p, 0, 4, ctx->own));
  CK(cudaStreamSynchronize(ctx->own));
  *out = ctx;
  return GG_OK;
}

gg_status gg_destroy(gg_context* ctx) {
  if (!ctx) return GG_E_INVALID;
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->own;
  cudaDeviceSynchronize();
  for (auto& sc : ctx->scenes) sc.free_all(ctx, s);
  for (auto& e : ctx->tev) cudaEventDestroy(e);
  for (Work* w : {&ctx->sw, &ctx->aw})
    for (int i = 0; i < Work::count; ++i) dev_free(ctx, w->all()[i], s);
  DevBuf* all[] = {&ctx->scene_table, &ctx->errflag, &ctx->valid_out,
                   &ctx->dbg_tc, &ctx->dbg_proj, &ctx->dbg_stile, &ctx->dbg_sz, &ctx->dbg_sgid,
                   &ctx->dbg_neval, &ctx->h_in[0], &ctx->h_in[1], &ctx->blur_vm, &ctx->blur_ids,
                   &ctx->blur_intr};
  for (DevBuf* b : all) dev_free(ctx, *b, s);
  cudaStreamSynchronize(s);
  cudaFreeHost(ctx->h_vcnt); cudaFreeHost(ctx->h_kcnt); cudaFreeHost(ctx->h_rbase);
  cudaFreeHost(ctx->h_kbase); cudaFreeHost(ctx->h_err);
  cudaFreeHost(ctx->h_ids); cudaFreeHost(ctx->h_perm); cudaFreeHost(ctx->h_groups); cudaFreeHost(ctx->h_blkbase);
  cudaFreeHost(ctx->h_vm);
  cudaEventDestroy(ctx->ev_copy);
  for (auto& e : ctx->h_done)
    if (e) cudaEventDestroy(e);
  cudaStreamDestroy(s);
  delete ctx;
  return GG_OK;
}

// Envs per pipeline pass when the caller did not fix it (gg_reserve chunk 0):
// the largest of 4096, 2048, 1024 whose workspace estimate -- records,
// depth-sort ping-pong and keys for `vis_frac` of the largest scene per env,
// ~100 B per visible record -- fits 80% of the device memory available to
// the context (free memory plus the workspace it already holds).  If a
// chunk's records or keys still do not fit, render_impl redoes that chunk in
// halves.  Fewer,
// larger passes have fewer kernel tails and host round trips (c3: 24.08k,
// 24.40k, 24.53k env-frames/s at 1024, 2048, 4096).
static int auto_chunk(gg_context* ctx, int E, double per_env_bytes, Work* reusable) {
  if (ctx->chunk > 0) return std::min(E, ctx->chunk);
  // cached per (E, estimate, workspace set): cudaMemGetInfo costs
  // milliseconds on a context holding tens of GB, too much for every render
  if (ctx->ac_E == E && ctx->ac_bytes == per_env_bytes && ctx->ac_set == reusable) return ctx->ac_chunk;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    cudaGetLastError();
    return std::min(E, 1024);
  }
  size_t held = 0;   // the workspace this path already holds (it is reused, not added)
  for (int i = 0; i < Work::count; ++i) held += reusable->all()[i].bytes;
  const double avail = 0.8 * (double)(fr + held);
  int c = std::min(E, 1024);
  for (int cand : {4096, 2048})
    if ((double)std::min(E, cand) * per_env_bytes <= avail) {
      c = std::min(E, cand);
      break;
    }
  ctx->ac_E = E;
  ctx->ac_bytes = per_env_bytes;
  ctx->ac_set = reusable;
  ctx->ac_chunk = c;
  return c;
}

// ~100 B of workspace per visible record (records 64 B, depth-sort ping-pong
// 16 B, keys ~2.2 x 4 B, order, histograms); the sync path budgets 30% of the
// largest scene visible per env
static double sync_env_bytes(const gg_context* ctx) { return (double)std::max(max_scene_n(ctx), 1) * 0.3 * 100.0; }

// Storage blocks per cull/project CTA: 1 when env groups are full (c3: 16
// envs of one view cell), up to 8 when they are small (c5: ~1.6 envs per
// scene), so a CTA's camera staging and launch are shared by more work.
static int blocks_per_cta(int ec, int ngroups) {
  const double avg = ngroups > 0 ? (double)ec / ngroups : ENV_GROUP;
  int b = 1;
  while (b < 8 && avg * b * 2 <= ENV_GROUP) b *= 2;
  return b;
}

// storage blocks per cull CTA: up to 16 (the CTA's block tests then run in
// one step and its camera staging is shared; measured at c3: 1 -> 4.64, 4 ->
// 4.11, 8 -> 3.98, 16 -> 3.96 ms), as long as the grid keeps >= 12 CTAs per SM
static int cull_blocks_per_cta(int ngroups, int nblk, int bpc) {
  static const int env = getenv("GG_CULL_BPC") ? atoi(getenv("GG_CULL_BPC")) : 0;   // A/B switch
  if (env > 0) return env;
  int b = 16;
  while (b > bpc && (long long)ngroups * ((nblk + b - 1) / b) < 148LL * 12) b /= 2;
  return std::max(b, bpc);
}

static gg_status upload_scene_table(gg_context* ctx) {
  const int n = (int)ctx->scenes.size();
  std::vector<DevScene> h(n);
  for (int i = 0; i < n; ++i) {
    h[i] = ctx->scenes[i].d;
    h[i].valid = ctx->scenes[i].live ? 1 : 0;
  }
  // capacity for SCENE_TABLE_MIN scenes up front: the table normally never
  // moves, so CUDA graphs captured over GG_ASYNC renders stay valid across
  // later gg_load_scene / gg_unload_scene calls (the table is read at replay)
  const void* before = ctx->scene_table.p;
  if (!ensure(ctx, ctx->scene_table, sizeof(DevScene) * std::max(n, SCENE_TABLE_MIN), ctx->own))
    return fail(ctx, GG_E_OOM, "scene table alloc");
  if (before && before != ctx->scene_table.p) ctx->async_ready = false;   // graphs over the old table are stale
  CK(cudaMemcpyAsync(ctx->scene_table.p, h.data(), sizeof(DevScene) * n, cudaMemcpyHostToDevice, ctx->own));
  CK(cudaStreamSynchronize(ctx->own));
  return GG_OK;
}

gg_status gg_load_scene(gg_context* ctx, int64_t n, int32_t d, const float* means, const float* scales,
                        const float* quats, const float* opac, const float* sh, int32_t* out_id) {
  if (!ctx) return GG_E_INVALID;
  if (!out_id || !means || !scales || !quats || !opac || !sh)
    return fail(ctx, GG_E_INVALID, "gg_load_scene: null pointer argument");
  if (n <= 0) return fail(ctx, GG_E_INVALID, "gg_load_scene: empty scene (n=%lld)", (long long)n);
  if (n > (int64_t)0x7fffff00) return fail(ctx, GG_E_UNSUPPORTED, "gg_load_scene: n too large");
  if (d < 0 || d > 3) return fail(ctx, GG_E_INVALID, "gg_load_scene: sh_degree %d not in 0..3", d);
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->own;
  const int K = (d + 1) * (d + 1);
  const size_t sz[5] = {(size_t)n * 3, (size_t)n * 3, (size_t)n * 4, (size_t)n, (size_t)n * K * 3};
  const float* src[5] = {means, scales, quats, opac, sh};
  DevBuf stage[5];
  const float* dsrc[5];
  for (int i = 0; i < 5; ++i) {
    if (is_device_ptr(src[i])) {
      dsrc[i] = src[i];
    } else {
      if (!ensure(ctx, stage[i], sz[i] * 4, s)) {
        for (auto& b : stage) dev_free(ctx, b, s);
        return fail(ctx, GG_E_OOM, "gg_load_scene: staging alloc");
      }
      CK(cudaMemcpyAsync(stage[i].p, src[i], sz[i] * 4, cudaMemcpyHostToDevice, s));
      dsrc[i] = P<float>(stage[i]);
    }
  }
  if (!ensure(ctx, ctx->valid_out, sizeof(ValidateOut), s)) return fail(ctx, GG_E_OOM, "alloc");
  CK(cudaMemsetAsync(ctx->valid_out.p, 0xff, sizeof(ValidateOut), s));
  launch_validate(n, K, dsrc[0], dsrc[1], dsrc[2], dsrc[3], dsrc[4], P<ValidateOut>(ctx->valid_out), s);
  ctx->launches++;
  ValidateOut vo;
  CK(cudaMemcpyAsync(&vo, ctx->valid_out.p, sizeof vo, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const unsigned long long NONE = ~0ULL;
  gg_status st = GG_OK;
  if (vo.nonfinite != NONE)
    st = fail(ctx, GG_E_NONFINITE, "gg_load_scene: non-finite value in record %llu", vo.nonfinite);
  else if (vo.bad_scale != NONE)
    st = fail(ctx, GG_E_INVALID, "gg_load_scene: scale <= 0 in record %llu", vo.bad_scale);
  else if (vo.bad_opacity != NONE)
    st = fail(ctx, GG_E_INVALID, "gg_load_scene: opacity outside [0,1] in record %llu", vo.bad_opacity);
  else if (vo.zero_quat != NONE)
    st = fail(ctx, GG_E_INVALID, "gg_load_scene: zero-norm quaternion in record %llu", vo.zero_quat);
  if (st != GG_OK) {
    for (auto& b : stage) dev_free(ctx, b, s);
    cudaStreamSynchronize(s);
    return st;
  }
  SceneSlot slot;
  const int sh_stride = d > 0 ? ((K * 3 + 3) / 4) * 4 : 0;
  const int64_t nblk = (n + PROJ_BLOCK - 1) / PROJ_BLOCK;
  bool ok = ensure(ctx, slot.pos_op, n * 16, s) && ensure(ctx, slot.cov_a, n * 16, s) &&
            ensure(ctx, slot.cov_b, n * 16, s) && ensure(ctx, slot.aux, n * 8, s) && ensure(ctx, slot.qmax, n * 4, s) &&
            ensure(ctx, slot.gid, n * 4, s) && ensure(ctx, slot.bbox, nblk * 32, s) &&
            (d == 0 || ensure(ctx, slot.sh, (size_t)n * sh_stride * 4, s));
  // spatial (Morton) storage order: scratch for the load-time sort
  const bool spatial = getenv("GG_NO_SPATIAL_ORDER") == nullptr;   // A/B switch (input order when set)
  DevBuf perm, tmp, hist, box;
  if (ok && spatial)
    ok = ensure(ctx, perm, n * 4, s) && ensure(ctx, tmp, n * 12, s) &&
         ensure(ctx, hist, (size_t)((n + 255) / 256) * 16 * 4, s) && ensure(ctx, box, 32, s);
  if (!ok) {
    for (auto& b : stage) dev_free(ctx, b, s);
    for (DevBuf* b : {&perm, &tmp, &hist, &box}) dev_free(ctx, *b, s);
    slot.free_all(ctx, s);
    return fail(ctx, GG_E_OOM, "gg_load_scene: out of device memory for %lld Gaussians", (long long)n);
  }
  if (spatial)
    ctx->launches += launch_spatial_order(n, dsrc[0], P<uint32_t>(box), P<uint32_t>(tmp), P<uint32_t>(hist),
                                          P<uint32_t>(perm), s);
  launch_pack(n, K, sh_stride, dsrc[0], dsrc[1], dsrc[2], dsrc[3], dsrc[4], spatial ? P<uint32_t>(perm) : nullptr,
              P<float4>(slot.pos_op), P<float4>(slot.cov_a), P<float4>(slot.cov_b), P<float2>(slot.aux),
              P<float>(slot.qmax), d > 0 ? P<float>(slot.sh) : nullptr, P<uint32_t>(slot.gid), s);
  launch_block_bounds((int)n, P<float4>(slot.pos_op), P<float2>(slot.aux), P<float4>(slot.bbox), s);
  ctx->launches += 2;
  CK(cudaGetLastError());
  for (auto& b : stage) dev_free(ctx, b, s);
  for (DevBuf* b : {&perm, &tmp, &hist, &box}) dev_free(ctx, *b, s);
  slot.d.pos_op = P<float4>(slot.pos_op);
  slot.d.cov_a = P<float4>(slot.cov_a);
  slot.d.cov_b = P<float4>(slot.cov_b);
  slot.d.aux = P<float2>(slot.aux);
  slot.d.qmax = P<float>(slot.qmax);
  slot.d.sh4 = d > 0 ? P<float4>(slot.sh) : nullptr;
  slot.d.gid = P<uint32_t>(slot.gid);
  slot.d.bbox = P<float4>(slot.bbox);
  slot.d.n = (int32_t)n;
  slot.d.degree = d;
  slot.d.sh_stride = sh_stride;
  slot.d.valid = 1;
  slot.live = true;
  // reuse a free id if any
  int id = -1;
  for (size_t i = 0; i < ctx->scenes.size(); ++i)
    if (!ctx->scenes[i].live) { id = (int)i; break; }
  if (id < 0) {
    id = (int)ctx->scenes.size();
    ctx->scenes.push_back(slot);
  } else {
    ctx->scenes[id] = slot;
  }
  gg_status us = upload_scene_table(ctx);
  if (us != GG_OK) return us;
  *out_id = id;
  return GG_OK;
}

gg_status gg_unload_scene(gg_context* ctx, int32_t id) {
  if (!ctx) return GG_E_INVALID;
  if (id < 0 || id >= (int)ctx->scenes.size() || !ctx->scenes[id].live)
    return fail(ctx, GG_E_BAD_SCENE, "gg_unload_scene: unknown scene id %d", id);
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  SceneSlot& sc = ctx->scenes[id];
  sc.free_all(ctx, ctx->own);
  sc.live = false;
  sc.d = DevScene{};
  return upload_scene_table(ctx);
}

gg_status gg_reserve(gg_context* ctx, int32_t max_envs, int32_t W, int32_t H, int32_t chunk) {
  if (!ctx) return GG_E_INVALID;
  if (max_envs <= 0 || W <= 0 || H <= 0 || chunk < 0) return fail(ctx, GG_E_INVALID, "gg_reserve: bad sizes");
  if (chunk > 0) ctx->chunk = chunk;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->own;
  const int ec = auto_chunk(ctx, max_envs, sync_env_bytes(ctx), &ctx->sw);
  const int nmax = std::max(max_scene_n(ctx), 1);
  const int nblk = (nmax + PROJ_BLOCK - 1) / PROJ_BLOCK;
  const int ntiles = ((W + TILE - 1) / TILE) * ((H + TILE - 1) / TILE);
  bool ok = ensure(ctx, ctx->sw.envc, sizeof(EnvConst) * max_envs, s) &&
            ensure(ctx, ctx->sw.flags, (size_t)ec * nblk * PROJ_WPB * 4, s) &&
            ensure(ctx, ctx->sw.blkcnt, (size_t)ec * nblk * 4, s) && ensure(ctx, ctx->sw.vcnt, ec * 4, s) &&
            ensure(ctx, ctx->sw.kcnt, ec * 8, s) && ensure(ctx, ctx->sw.rbase, ec * 8, s) &&
            ensure(ctx, ctx->sw.kbase, ec * 8, s) && ensure(ctx, ctx->sw.ranges, (size_t)ec * ntiles * 8, s) &&
            ensure(ctx, ctx->sw.counters, (size_t)max_envs * 32, s) && ensure_host(ctx, ec);
  CK(cudaStreamSynchronize(s));
  return ok ? GG_OK : fail(ctx, GG_E_OOM, "gg_reserve: allocation failed");
}

gg_status gg_set_timing(gg_context* ctx, int32_t en) {
  if (!ctx) return GG_E_INVALID;
  ctx->timing = en != 0;
  return GG_OK;
}

static gg_status resolve_timing(gg_context* ctx) {
  if (ctx->t_nchunks == 0) return GG_OK;
  float ms[NSTAGE] = {0, 0, 0, 0, 0};
  CK(cudaEventSynchronize(ctx->tev[ctx->t_nchunks * (NSTAGE + 1) - 1]));
  for (int c = 0; c < ctx->t_nchunks; ++c)
    for (int k = 0; k < NSTAGE; ++k) {
      float x = 0;
      CK(cudaEventElapsedTime(&x, ctx->tev[c * (NSTAGE + 1) + k], ctx->tev[c * (NSTAGE + 1) + k + 1]));
      ms[k] += x;
    }
  for (int k = 0; k < NSTAGE; ++k) ctx->stage_ms[k] = ms[k];
  ctx->t_nchunks = 0;
  return GG_OK;
}

gg_status gg_get_stage_ms(gg_context* ctx, float* out3) {
  if (!ctx || !out3) return GG_E_INVALID;
  gg_status st = resolve_timing(ctx);
  if (st != GG_OK) return st;
  out3[0] = ctx->stage_ms[0] + ctx->stage_ms[1];
  out3[1] = ctx->stage_ms[2] + ctx->stage_ms[3];
  out3[2] = ctx->stage_ms[4];
  return GG_OK;
}

gg_status gg_get_stage_times(gg_context* ctx, float* out, int32_t n) {
  if (!ctx || !out || n < 1 || n > NSTAGE) return GG_E_INVALID;
  gg_status st = resolve_timing(ctx);
  if (st != GG_OK) return st;
  for (int i = 0; i < n; ++i) out[i] = ctx->stage_ms[i];
  return GG_OK;
}

// Core pipeline.  `after_chunk` (optional) is invoked after each chunk's
// rasterize is enqueued (used by gg_render_host to stream outputs out).
// Called after the rasterisation of processing positions [p0, p0 + n) has
// been enqueued on the render stream (ctx->h_perm maps positions to caller
// env indices).
typedef gg_status (*chunk_cb)(gg_context*, int p0, int n, void* user);
constexpr int HOST_COPY_SLICE = 128;   // envs per raster launch when frames stream to the host

static uint32_t f32_bits(float x) {
  uint32_t b;
  memcpy(&b, &x, 4);
  return b;
}

// depth-sort passes: keys are z bits - bits(near) in (0, bits(far) - bits(near)]
static int depth_passes_for(float near_p, float far_p) { return depth_passes(f32_bits(far_p) - f32_bits(near_p)); }

// The NSTAGE + 1 timing events of chunk c of the current render (created on
// demand; events are never created or recorded unless timing is enabled).
static cudaEvent_t* chunk_events(gg_context* ctx, int c) {
  const size_t need = (size_t)(c + 1) * (NSTAGE + 1);
  while (ctx->tev.size() < need) {
    cudaEvent_t ev = nullptr;
    if (cudaEventCreate(&ev) != cudaSuccess) return nullptr;
    ctx->tev.push_back(ev);
  }
  return ctx->tev.data() + (size_t)c * (NSTAGE + 1);
}

#define TREC(k)                                                                  \
  do {                                                                           \
    if (tev) CK(cudaEventRecord(tev[k], s));                                     \
  } while (0)

// Motion blur fused into the raster (gg_render_blur): the E cameras are the
// Kc consecutive sample cameras of E / Kc envs; outputs are per env.
struct BlurSpec {
  int K, Kc, dk;
};

static gg_status render_impl(gg_context* ctx, int32_t E, const int32_t* scene_ids, const float* viewmats,
                             const float* intr, int32_t W, int32_t H, const gg_render_opts* opts_in,
                             void* rgb, float* depth, float* alpha, cudaStream_t s, chunk_cb cb,
                             void* cb_user, const BlurSpec* blur = nullptr) {
  gg_render_opts opts;
  if (opts_in) opts = *opts_in; else gg_default_opts(&opts);
  if (E <= 0 || W <= 0 || H <= 0) return fail(ctx, GG_E_INVALID, "gg_render: n_envs/width/height must be > 0");
  if (!scene_ids || !viewmats || !intr) return fail(ctx, GG_E_INVALID, "gg_render: null input pointer");
  if (opts.rgb_format != 0 && opts.rgb_format != 1) return fail(ctx, GG_E_INVALID, "gg_render: rgb_format");
  if (!(opts.near_plane > 0.f) || !(opts.far_plane > opts.near_plane))
    return fail(ctx, GG_E_INVALID, "gg_render: need 0 < near < far");
  if (opts.sh_degree > 3) return fail(ctx, GG_E_INVALID, "gg_render: sh_degree > 3");
  const int TX = (W + TILE - 1) / TILE, TY = (H + TILE - 1) / TILE;
  const int ntiles = TX * TY;
  if (ntiles > MAX_TILES || W > 65535 || H > 65535)
    return fail(ctx, GG_E_UNSUPPORTED, "gg_render: %dx%d needs %d tiles > %d", W, H, ntiles, MAX_TILES);
  if (ctx->scenes.empty()) return fail(ctx, GG_E_BAD_SCENE, "gg_render: no scene loaded");
  CK(cudaSetDevice(ctx->device));

  RenderParams rp;
  rp.W = W; rp.H = H; rp.TX = TX; rp.TY = TY; rp.ntiles = ntiles;
  rp.near_p = opts.near_plane; rp.far_p = opts.far_plane;
  rp.bg[0] = opts.background[0]; rp.bg[1] = opts.background[1]; rp.bg[2] = opts.background[2];
  rp.rgb_format = opts.rgb_format;
  rp.tight = (opts.flags & (GG_TIGHT_TILES | GG_ELLIPSE_TILES)) != 0;
  rp.ellipse = (opts.flags & GG_ELLIPSE_TILES) != 0;
  rp.color = rgb != nullptr;
  rp.blur_k = blur ? blur->K : 0;
  rp.blur_kc = blur ? blur->Kc : 0;
  rp.blur_dk = blur ? blur->dk : 0;
  const bool counters = (opts.flags & GG_COUNTERS) != 0 && !blur;
  const bool keep = (opts.flags & GG_KEEP_INTERMEDIATES) != 0 && opts.debug_env >= 0 && opts.debug_env < E && !blur;

  const int nmax = std::max(max_scene_n(ctx), 1);
  const int nblk = (nmax + PROJ_BLOCK - 1) / PROJ_BLOCK;
  const int nwords = nblk * (PROJ_BLOCK / 32);
  int chunk = auto_chunk(ctx, E, sync_env_bytes(ctx), &ctx->sw);
  if (cb) chunk = std::min(chunk, 1024);   // host outputs: finer chunks interleave the frame copies with compute
  ctx->last_chunk = chunk;
  if (blur) chunk = std::max(blur->Kc, chunk / blur->Kc * blur->Kc);   // an env's samples never straddle chunks

  if (!ensure(ctx, ctx->sw.envc, sizeof(EnvConst) * E, s) || !ensure(ctx, ctx->sw.perm, (size_t)E * 4, s) ||
      !ensure(ctx, ctx->sw.groups, sizeof(EnvGroup) * (size_t)chunk, s) ||
      !ensure(ctx, ctx->sw.flags, (size_t)chunk * nwords * 4, s) ||
      !ensure(ctx, ctx->sw.blkcnt, (size_t)chunk * nblk * 4, s) || !ensure(ctx, ctx->sw.vcnt, chunk * 4, s) ||
      !ensure(ctx, ctx->sw.kcnt, chunk * 8, s) || !ensure(ctx, ctx->sw.rbase, chunk * 8, s) ||
      !ensure(ctx, ctx->sw.kbase, chunk * 8, s) || !ensure(ctx, ctx->sw.ranges, (size_t)chunk * ntiles * 8, s) ||
      !ensure_host(ctx, std::max(E, chunk)) || (counters && !ensure(ctx, ctx->sw.counters, (size_t)E * 32, s)))
    return fail(ctx, GG_E_OOM, "gg_render: workspace allocation failed");
  if (counters) {
    CK(cudaMemsetAsync(ctx->sw.counters.p, 0, (size_t)E * 32, s));
    ctx->last_counters = &ctx->sw.counters;
  }
  CK(cudaMemsetAsync(ctx->errflag.p, 0, 4, s));

  // Processing order of the envs (outputs are still written at the caller's
  // env index, EnvConst.out_index, and every env's result depends only on its
  // own camera and scene, so the order changes no output bit): envs bound to
  // one scene become contiguous, so the projection kernels share each
  // Gaussian load across a group of <= 16 envs; inside a scene, envs are
  // ordered by view direction (a cube-map face of the forward axis, 2 x 2
  // cells per face) and then by the Morton code of the camera centre, so the
  // envs of a group look at the same storage blocks: whole (group, block)
  // tiles of the cull then fail the block test together and the projection's
  // pair lists get denser (spatial chunk culling).  With
  // host outputs (gg_render_host) the order is first by windows of
  // HOST_COPY_SLICE caller envs, so each raster slice's frames are one
  // contiguous range of the caller's buffer (one copy per slice).
  ctx->launches += launch_copy_words(ctx->h_ids, scene_ids, (size_t)E * 4, s);
  // (not for blur: an env's Kc sample cameras must stay consecutive)
  const bool view_order = getenv("GG_NO_ENV_ORDER") == nullptr && !blur;   // A/B switch
  if (view_order) ctx->launches += launch_copy_words(ctx->h_vm, viewmats, (size_t)E * 64, s);
  CK(cudaStreamSynchronize(s));
  const int nsc = (int)ctx->scenes.size();
  auto key = [&](int e) {
    const int id = ctx->h_ids[e];
    return (id < 0 || id >= nsc || !ctx->scenes[id].live) ? -1 : id;
  };
  std::vector<int32_t> order(E);
  for (int e = 0; e < E; ++e) order[e] = e;
  std::vector<uint32_t> vkey(view_order ? E : 0);
  if (view_order) {
    float lo[3] = {1e30f, 1e30f, 1e30f}, hi[3] = {-1e30f, -1e30f, -1e30f};
    std::vector<float> cc((size_t)E * 3);
    for (int e = 0; e < E; ++e) {
      const float* V = ctx->h_vm + (size_t)e * 16;
      for (int k = 0; k < 3; ++k) {
        const float c = -(V[0 * 4 + k] * V[3] + V[1 * 4 + k] * V[7] + V[2 * 4 + k] * V[11]);
        cc[(size_t)e * 3 + k] = std::isfinite(c) ? c : 0.f;
        lo[k] = std::min(lo[k], cc[(size_t)e * 3 + k]);
        hi[k] = std::max(hi[k], cc[(size_t)e * 3 + k]);
      }
    }
    auto spread = [](uint32_t x) {   // 4 bits -> every third bit
      uint32_t r = 0;
      for (int b = 0; b < 4; ++b) r |= ((x >> b) & 1u) << (3 * b);
      return r;
    };
    for (int e = 0; e < E; ++e) {
      const float* F = ctx->h_vm + (size_t)e * 16 + 8;   // forward axis (row 2 of R) in world coordinates
      int ax = 0;
      for (int k = 1; k < 3; ++k)
        if (std::fabs(F[k]) > std::fabs(F[ax])) ax = k;
      const float m = std::fabs(F[ax]) > 0.f ? std::fabs(F[ax]) : 1.f;
      const float a = F[(ax + 1) % 3] / m, b = F[(ax + 2) % 3] / m;   // in [-1, 1] on the face
      const uint32_t face = (uint32_t)(2 * ax + (F[ax] < 0.f));
      const uint32_t cell = (a >= 0.f ? 1u : 0u) | (b >= 0.f ? 2u : 0u);
      uint32_t pos = 0;
      for (int k = 0; k < 3; ++k) {
        const float ext = hi[k] - lo[k];
        const uint32_t qk = ext > 0.f ? (uint32_t)std::min(15.f, std::max(0.f, (cc[(size_t)e * 3 + k] - lo[k]) / ext * 16.f)) : 0u;
        pos |= spread(qk) << k;
      }
      vkey[e] = ((face * 4 + cell) << 12) | pos;
    }
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    if (cb && a / HOST_COPY_SLICE != b / HOST_COPY_SLICE) return a / HOST_COPY_SLICE < b / HOST_COPY_SLICE;
    const int ka = key(a), kb = key(b);
    if (ka != kb) return ka < kb;
    return view_order && vkey[a] < vkey[b];
  });
  int dbg_pos = -1;
  for (int p = 0; p < E; ++p) {
    ctx->h_perm[p] = order[p];
    if (keep && order[p] == opts.debug_env) dbg_pos = p;
  }
  ctx->launches += launch_copy_words(ctx->sw.perm.p, ctx->h_perm, (size_t)E * 4, s);
  launch_setup_envs(E, P<int32_t>(ctx->sw.perm), scene_ids, viewmats, intr, P<DevScene>(ctx->scene_table), nsc, W, H,
                    opts.sh_degree, P<EnvConst>(ctx->sw.envc), P<uint32_t>(ctx->errflag), s);
  ctx->launches++;
  CK(cudaGetLastError());

  if (!ctx->t_append) ctx->t_nchunks = 0;
  int cidx = ctx->t_nchunks;
  for (int e0 = 0, ec = 0; e0 < E; e0 += ec, ++cidx) {
    cudaEvent_t* tev = ctx->timing ? chunk_events(ctx, cidx) : nullptr;
    if (ctx->timing && !tev) return fail(ctx, GG_E_CUDA, "gg_render: timing events");
    ec = std::min(chunk, E - e0);
    if (cb && chunk >= 64) {
      // host path: a short first chunk gets frames onto the copy engine early,
      // a short last chunk leaves little of the copy backlog after the render
      const int q = chunk / 4, rem = E - e0;
      if (e0 == 0 && rem > q) ec = q;
      else if (rem > q && rem <= chunk + q) ec = rem - q;
    }
    // env groups: runs of one scene, <= ENV_GROUP envs
    int ngroups = 0, max_deg = 0;
    for (int i = 0; i < ec;) {
      const int k0 = key(order[e0 + i]);
      int j = i + 1;
      while (j < ec && j - i < ENV_GROUP && key(order[e0 + j]) == k0) ++j;
      ctx->h_groups[ngroups].elo = i;
      ctx->h_groups[ngroups].cnt = j - i;
      ++ngroups;
      if (k0 >= 0) {
        const int d = ctx->scenes[k0].d.degree;
        max_deg = std::max(max_deg, opts.sh_degree < 0 ? d : std::min(d, opts.sh_degree));
      }
      i = j;
    }
    ctx->launches += launch_copy_words(ctx->sw.groups.p, ctx->h_groups, sizeof(EnvGroup) * ngroups, s);
    ChunkWS ws{};
    ws.flags = P<uint32_t>(ctx->sw.flags);
    ws.blkcnt = P<uint32_t>(ctx->sw.blkcnt);
    ws.vcnt = P<uint32_t>(ctx->sw.vcnt);
    ws.kcnt = P<unsigned long long>(ctx->sw.kcnt);
    ws.rec_base = P<uint64_t>(ctx->sw.rbase);
    ws.k_base = P<uint64_t>(ctx->sw.kbase);
    ws.ranges = P<uint2>(ctx->sw.ranges);
    ws.zbase = f32_bits(opts.near_plane);
    ws.nwords = nwords;
    ws.nblk = nblk;
    ws.ec = ec;
    const EnvGroup* groups = P<EnvGroup>(ctx->sw.groups);
    TREC(0);
    // K1a + K2
    // storage blocks per CTA: small env groups share a CTA's setup over several blocks
    const int bpc = blocks_per_cta(ec, ngroups);
    launch_cull_count(e0, ngroups, nblk, cull_blocks_per_cta(ngroups, nblk, bpc), groups, P<EnvConst>(ctx->sw.envc), P<DevScene>(ctx->scene_table), rp, ws,
                      s);
    launch_scan_blocks(ec, nblk, ws.blkcnt, ws.vcnt, s);
    ctx->launches += 2;
    CK(cudaGetLastError());
    TREC(1);
    ctx->launches += launch_copy_words(ctx->h_vcnt, ws.vcnt, ec * 4, s);
    CK(cudaStreamSynchronize(s));
    uint64_t V = 0;
    for (int i = 0; i < ec; ++i) { ctx->h_rbase[i] = V; V += ctx->h_vcnt[i]; }
    if (!ensure(ctx, ctx->sw.rec0, V * 16, s) || !ensure(ctx, ctx->sw.rec1, V * 16, s) ||
        !ensure(ctx, ctx->sw.rec2, V * 16, s) || !ensure(ctx, ctx->sw.rect, V * 8, s) ||
        !ensure(ctx, ctx->sw.zkey, V * 4, s) || !ensure(ctx, ctx->sw.gid, V * 4, s) ||
        (rp.ellipse && !ensure(ctx, ctx->sw.rmask, V * 4 + 4, s)) ||
        (keep && !ensure(ctx, ctx->sw.dconic, V * 16, s)) ||
        !ensure(ctx, ctx->sw.dk0, V * 8, s) || !ensure(ctx, ctx->sw.dk1, V * 8, s) ||
        !ensure(ctx, ctx->sw.dv0, V * 4, s)) {
      const int unit = blur ? blur->Kc : 64;
      if (ec >= 2 * unit) {   // too many records for the memory left: redo this chunk in halves
        chunk = std::max(unit, (ec / 2) / unit * unit);
        ec = 0;
        --cidx;
        continue;
      }
      return fail(ctx, GG_E_OOM, "gg_render: record workspace (%llu records) allocation failed",
                  (unsigned long long)V);
    }
    ctx->launches += launch_copy_words(ctx->sw.rbase.p, ctx->h_rbase, ec * 8, s);
    CK(cudaMemsetAsync(ws.kcnt, 0, ec * 8, s));
    ws.rec0 = P<float4>(ctx->sw.rec0); ws.rec1 = P<float4>(ctx->sw.rec1); ws.rec2 = P<float4>(ctx->sw.rec2);
    ws.rect = P<uint2>(ctx->sw.rect); ws.zkey = P<uint32_t>(ctx->sw.zkey);
    ws.rmask = rp.ellipse ? P<uint32_t>(ctx->sw.rmask) : nullptr;
    ws.gid = P<uint32_t>(ctx->sw.gid);
    ws.dconic = keep ? P<float4>(ctx->sw.dconic) : nullptr;
    ws.dp0 = P<uint64_t>(ctx->sw.dk0); ws.dp1 = P<uint64_t>(ctx->sw.dk1); ws.order = P<uint32_t>(ctx->sw.dv0);
    // K1b
    launch_project(e0, ngroups, nblk, bpc, max_deg, groups, P<EnvConst>(ctx->sw.envc), P<DevScene>(ctx->scene_table), rp,
                   ws, s);
    ctx->launches++;
    CK(cudaGetLastError());
    ctx->launches += launch_copy_words(ctx->h_kcnt, ws.kcnt, ec * 8, s);
    TREC(2);
    CK(cudaStreamSynchronize(s));
    uint64_t K = 0;
    for (int i = 0; i < ec; ++i) { ctx->h_kbase[i] = K; K += ctx->h_kcnt[i]; }
    if (!blur) {   // calibration record for gg_reserve_async (negative max_visible_frac)
      if (ctx->cal_W != W || ctx->cal_H != H) {
        ctx->cal_vmean = ctx->cal_kmean = 0.0;
        ctx->cal_vmax = ctx->cal_kmax = 0;
        ctx->cal_W = W; ctx->cal_H = H;
      }
      ctx->cal_vmean = std::max(ctx->cal_vmean, (double)V / ec);
      ctx->cal_kmean = std::max(ctx->cal_kmean, (double)K / ec);
      for (int i = 0; i < ec; ++i) {
        ctx->cal_vmax = std::max<uint64_t>(ctx->cal_vmax, ctx->h_vcnt[i]);
        ctx->cal_kmax = std::max<uint64_t>(ctx->cal_kmax, ctx->h_kcnt[i]);
      }
    }
    for (int i = 0; i < ec; ++i)
      if (ctx->h_kcnt[i] > 0xffffffffull)
        return fail(ctx, GG_E_CAPACITY, "gg_render: env %d has %llu tile keys (>= 2^32)", ctx->h_perm[e0 + i],
                    (unsigned long long)ctx->h_kcnt[i]);
    if (!ensure(ctx, ctx->sw.sorted, K * 4, s)) {
      const int unit = blur ? blur->Kc : 64;
      if (ec >= 2 * unit) {   // too many keys for the memory left: redo this chunk in halves
        chunk = std::max(unit, (ec / 2) / unit * unit);
        ec = 0;
        --cidx;
        continue;
      }
      return fail(ctx, GG_E_OOM, "gg_render: key workspace (%llu keys) allocation failed", (unsigned long long)K);
    }
    ctx->launches += launch_copy_words(ctx->sw.kbase.p, ctx->h_kbase, ec * 8, s);
    ws.sorted = P<uint32_t>(ctx->sw.sorted);
#ifdef GG_CHECK_PROTOCOLS
    CK(cudaMemsetAsync(ws.sorted, 0xff, K * 4, s));   // placement asserts each slot is written once
#endif
    // K3-K5: sort blocks of sort_block_size() records, never straddling an env
    uint32_t nb = 0;
    for (int i = 0; i < ec; ++i) { ctx->h_blkbase[i] = nb; nb += sort_blocks(ctx->h_vcnt[i]); }
    ctx->h_blkbase[ec] = nb;
    const int passes = depth_passes_for(opts.near_plane, opts.far_plane);
    if (!ensure(ctx, ctx->sw.blkbase, (size_t)(ec + 1) * 4, s) || !ensure(ctx, ctx->sw.blkenv, (size_t)nb * 4 + 4, s) ||
        !ensure(ctx, ctx->sw.ghist, (size_t)nb * sort_ghist_words() * 4, s) ||
        !ensure(ctx, ctx->sw.thist, (size_t)nb * ntiles * 4, s)) {
      const int unit = blur ? blur->Kc : 64;
      if (ec >= 2 * unit) {   // redo this chunk in halves
        chunk = std::max(unit, (ec / 2) / unit * unit);
        ec = 0;
        --cidx;
        continue;
      }
      return fail(ctx, GG_E_OOM, "gg_render: sort workspace allocation failed");
    }
    ctx->launches += launch_copy_words(ctx->sw.blkbase.p, ctx->h_blkbase, (size_t)(ec + 1) * 4, s);
    ctx->launches += launch_sort_bin(ec, nb, P<uint32_t>(ctx->sw.blkbase), P<uint32_t>(ctx->sw.blkenv), passes, rp, ws,
                                     P<uint32_t>(ctx->sw.ghist),
                                     P<uint32_t>(ctx->sw.thist), s, false, nullptr, tev ? tev[3] : nullptr);
    CK(cudaGetLastError());
    TREC(4);
    // K6
    const int dbg_eloc = (dbg_pos >= e0 && dbg_pos < e0 + ec) ? dbg_pos - e0 : -1;
    int32_t* dbg_neval = nullptr;
    if (dbg_eloc >= 0 && counters) {
      if (!ensure(ctx, ctx->dbg_neval, (size_t)W * H * 4, s)) return fail(ctx, GG_E_OOM, "debug alloc");
      dbg_neval = P<int32_t>(ctx->dbg_neval);
    }
    if (cb) {
      // host path: raster in slices, each slice's frames start copying to the
      // host while the next slice renders (only the last slice's copy is exposed)
      for (int s0 = 0; s0 < ec; s0 += HOST_COPY_SLICE) {
        const int n = std::min(HOST_COPY_SLICE, ec - s0);
        ChunkWS wss = ws;
        wss.ranges = ws.ranges + (size_t)s0 * ntiles;
        wss.rec_base = ws.rec_base + s0;
        wss.k_base = ws.k_base + s0;
        wss.vcnt = ws.vcnt + s0;
        wss.kcnt = ws.kcnt + s0;
        const int dl = (dbg_eloc >= s0 && dbg_eloc < s0 + n) ? dbg_eloc - s0 : -1;
        launch_raster(e0 + s0, n, P<EnvConst>(ctx->sw.envc), rp, wss, rgb, depth, alpha, counters,
                      counters ? P<unsigned long long>(ctx->sw.counters) : nullptr, dl >= 0 ? dbg_neval : nullptr, dl,
                      s);
        ctx->launches++;
        CK(cudaGetLastError());
        gg_status cs = cb(ctx, e0 + s0, n, cb_user);
        if (cs != GG_OK) return cs;
      }
    } else {
      launch_raster(e0, ec, P<EnvConst>(ctx->sw.envc), rp, ws, rgb, depth, alpha, counters,
                    counters ? P<unsigned long long>(ctx->sw.counters) : nullptr, dbg_neval, dbg_eloc, s);
      ctx->launches++;
      CK(cudaGetLastError());
    }
    TREC(5);
    if (dbg_eloc >= 0) {
      // K8: snapshot the debug env's integer artefacts to host
      const uint32_t Vd = ctx->h_vcnt[dbg_eloc], Kd = (uint32_t)ctx->h_kcnt[dbg_eloc];
      const uint64_t rb = ctx->h_rbase[dbg_eloc], kb = ctx->h_kbase[dbg_eloc];
      const int n_all = nmax;
      if (!ensure(ctx, ctx->dbg_tc, (size_t)n_all * 4, s) || !ensure(ctx, ctx->dbg_proj, (size_t)n_all * 64, s) ||
          !ensure(ctx, ctx->dbg_stile, (size_t)Kd * 4 + 4, s) || !ensure(ctx, ctx->dbg_sz, (size_t)Kd * 4 + 4, s) ||
          !ensure(ctx, ctx->dbg_sgid, (size_t)Kd * 4 + 4, s))
        return fail(ctx, GG_E_OOM, "debug alloc");
      CK(cudaMemsetAsync(ctx->dbg_tc.p, 0, (size_t)n_all * 4, s));
      CK(cudaMemsetAsync(ctx->dbg_proj.p, 0, (size_t)n_all * 64, s));
      launch_debug_records(Vd, rb, ws, P<int32_t>(ctx->dbg_tc), P<float>(ctx->dbg_proj), s);
      launch_debug_sorted(ntiles, ws.ranges + (size_t)dbg_eloc * ntiles, kb, rb, ws, P<int32_t>(ctx->dbg_stile),
                          P<uint32_t>(ctx->dbg_sz), P<int32_t>(ctx->dbg_sgid), s);
      ctx->launches += 2;
      CK(cudaGetLastError());
      EnvConst hc;
      CK(cudaMemcpyAsync(&hc, P<EnvConst>(ctx->sw.envc) + dbg_pos, sizeof hc, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      const int nn = std::max(hc.n, 0);
      ctx->d_tc.resize(nn); ctx->d_proj.resize((size_t)nn * 16);
      ctx->d_stile.resize(Kd); ctx->d_sz.resize(Kd); ctx->d_sgid.resize(Kd);
      ctx->d_ranges.resize((size_t)ntiles * 2);
      CK(cudaMemcpy(ctx->d_tc.data(), ctx->dbg_tc.p, (size_t)nn * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ctx->d_proj.data(), ctx->dbg_proj.p, (size_t)nn * 64, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ctx->d_stile.data(), ctx->dbg_stile.p, (size_t)Kd * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ctx->d_sz.data(), ctx->dbg_sz.p, (size_t)Kd * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ctx->d_sgid.data(), ctx->dbg_sgid.p, (size_t)Kd * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(ctx->d_ranges.data(), ws.ranges + (size_t)dbg_eloc * ntiles, (size_t)ntiles * 8,
                    cudaMemcpyDeviceToHost));
      ctx->d_counters[2] = Vd;
      ctx->d_counters[3] = Kd;
      if (counters) {
        unsigned long long c2[2];
        CK(cudaMemcpy(c2, P<unsigned long long>(ctx->sw.counters) + (size_t)opts.debug_env * 4, 16,
                      cudaMemcpyDeviceToHost));
        ctx->d_counters[0] = (int64_t)c2[0];
        ctx->d_counters[1] = (int64_t)c2[1];
        ctx->d_neval.resize((size_t)W * H);
        CK(cudaMemcpy(ctx->d_neval.data(), ctx->dbg_neval.p, (size_t)W * H * 4, cudaMemcpyDeviceToHost));
      } else {
        ctx->d_counters[0] = ctx->d_counters[1] = -1;
        ctx->d_neval.clear();
      }
    }
  }
  if (ctx->timing) ctx->t_nchunks = cidx;
  ctx->last_E = E;
  ctx->launches += launch_copy_words(ctx->h_err, ctx->errflag.p, 4, s);
  CK(cudaStreamSynchronize(s));
  if (*ctx->h_err & ERR_BAD_SCENE) return fail(ctx, GG_E_BAD_SCENE, "gg_render: an env is bound to an unknown scene id");
  return GG_OK;
}


// ---------------------------------------------------------------------------
// Sync-free mode (GG_ASYNC): fixed, pre-reserved workspace; every offset
// table is built on the device (async.cu), grids have fixed sizes, envs are
// taken in caller order in fixed groups of 16 (mixed scenes allowed), the
// number of depth passes follows from [near, far].  No host synchronisation
// and no allocation: the call can be captured in a CUDA graph.  Capacity
// overflow marks the chunk invalid and raises a sticky GG_E_CAPACITY.

static gg_status render_async(gg_context* ctx, int32_t E, const int32_t* scene_ids, const float* viewmats,
                              const float* intr, int32_t W, int32_t H, const gg_render_opts& opts, void* rgb,
                              float* depth, float* alpha, cudaStream_t s) {
  if (!ctx->async_ready) return fail(ctx, GG_E_INVALID, "GG_ASYNC: call gg_reserve_async first (again after the scene table moved)");
  if (E > ctx->a_max_envs || W != ctx->a_W || H != ctx->a_H)
    return fail(ctx, GG_E_CAPACITY, "GG_ASYNC: render (%d envs, %dx%d) exceeds the reservation (%d, %dx%d)", E, W, H,
                ctx->a_max_envs, ctx->a_W, ctx->a_H);
  if (opts.flags & GG_KEEP_INTERMEDIATES) return fail(ctx, GG_E_UNSUPPORTED, "GG_ASYNC: no intermediates");
  if ((opts.flags & GG_COUNTERS) && ctx->aw.counters.bytes < (size_t)E * 32)
    return fail(ctx, GG_E_CAPACITY, "GG_ASYNC: counters not reserved");
  const int TX = (W + TILE - 1) / TILE, TY = (H + TILE - 1) / TILE;
  RenderParams rp;
  rp.W = W; rp.H = H; rp.TX = TX; rp.TY = TY; rp.ntiles = TX * TY;
  rp.near_p = opts.near_plane; rp.far_p = opts.far_plane;
  rp.bg[0] = opts.background[0]; rp.bg[1] = opts.background[1]; rp.bg[2] = opts.background[2];
  rp.rgb_format = opts.rgb_format;
  rp.tight = (opts.flags & (GG_TIGHT_TILES | GG_ELLIPSE_TILES)) != 0;
  rp.blur_k = rp.blur_kc = rp.blur_dk = 0;
  rp.ellipse = (opts.flags & GG_ELLIPSE_TILES) != 0;
  rp.color = rgb != nullptr;
  const bool counters = (opts.flags & GG_COUNTERS) != 0;
  const int chunk = ctx->a_chunk, nblk = ctx->a_nblk, nwords = nblk * (PROJ_BLOCK / 32);
  if (nblk < (max_scene_n(ctx) + PROJ_BLOCK - 1) / PROJ_BLOCK)
    return fail(ctx, GG_E_CAPACITY, "GG_ASYNC: a scene larger than at gg_reserve_async time was loaded");
  const int passes = depth_passes_for(opts.near_plane, opts.far_plane);
  uint32_t* err = P<uint32_t>(ctx->errflag);
  uint32_t* ok = P<uint32_t>(ctx->aw.okflag);
  if (counters) {
    CK(cudaMemsetAsync(ctx->aw.counters.p, 0, (size_t)E * 32, s));
    ctx->last_counters = &ctx->aw.counters;
  }
  // envs in (scene, view) order on the device (the sync path sorts on the host)
  static const bool no_order = getenv("GG_NO_ENV_ORDER") != nullptr;   // A/B switch
  const bool ordered = !no_order && launch_env_order(E, scene_ids, viewmats, (int)ctx->scenes.size(),
                                                    P<DevScene>(ctx->scene_table), P<int32_t>(ctx->aw.perm), s);
  ctx->launches += ordered ? 1 : 0;
  launch_setup_envs(E, ordered ? P<int32_t>(ctx->aw.perm) : nullptr, scene_ids, viewmats, intr,
                    P<DevScene>(ctx->scene_table), (int)ctx->scenes.size(), W, H, opts.sh_degree,
                    P<EnvConst>(ctx->aw.envc), err, s);
  ctx->launches++;
  const int nchunks = (E + chunk - 1) / chunk;
  ctx->last_chunk = chunk;
  ctx->t_nchunks = 0;
  for (int c = 0; c < nchunks; ++c) {
    cudaEvent_t* tev = ctx->timing ? chunk_events(ctx, c) : nullptr;
    if (ctx->timing && !tev) return fail(ctx, GG_E_CUDA, "gg_render: timing events");
    const int e0 = c * chunk, ec = std::min(chunk, E - e0);
    const int ngroups = (ec + ENV_GROUP - 1) / ENV_GROUP;
    ChunkWS ws{};
    ws.flags = P<uint32_t>(ctx->aw.flags);
    ws.blkcnt = P<uint32_t>(ctx->aw.blkcnt);
    ws.vcnt = P<uint32_t>(ctx->aw.vcnt);
    ws.kcnt = P<unsigned long long>(ctx->aw.kcnt);
    ws.rec_base = P<uint64_t>(ctx->aw.rbase);
    ws.k_base = P<uint64_t>(ctx->aw.kbase);
    ws.rec0 = P<float4>(ctx->aw.rec0); ws.rec1 = P<float4>(ctx->aw.rec1); ws.rec2 = P<float4>(ctx->aw.rec2);
    ws.rect = P<uint2>(ctx->aw.rect); ws.zkey = P<uint32_t>(ctx->aw.zkey); ws.gid = P<uint32_t>(ctx->aw.gid);
    ws.rmask = rp.ellipse ? P<uint32_t>(ctx->aw.rmask) : nullptr;
    ws.zbase = f32_bits(opts.near_plane);
    ws.dp0 = P<uint64_t>(ctx->aw.dk0); ws.dp1 = P<uint64_t>(ctx->aw.dk1); ws.order = P<uint32_t>(ctx->aw.dv0);
    ws.sorted = P<uint32_t>(ctx->aw.sorted);
    ws.ranges = P<uint2>(ctx->aw.ranges);
    ws.ok = ok;
    ws.nwords = nwords;
    ws.nblk = nblk;
    ws.ec = ec;
    TREC(0);
    CK(cudaMemsetAsync(ws.kcnt, 0, ec * 8, s));
    CK(cudaMemsetAsync(ok, 0x01, 4, s));
    launch_cull_count(e0, ngroups, nblk, cull_blocks_per_cta(ngroups, nblk, 1), nullptr, P<EnvConst>(ctx->aw.envc),
                      P<DevScene>(ctx->scene_table), rp, ws, s);
    launch_scan_blocks(ec, nblk, ws.blkcnt, ws.vcnt, s);
    launch_tables_v(ec, ws.vcnt, P<uint64_t>(ctx->aw.rbase), ctx->a_vcap, ok, err, s);
    TREC(1);
    launch_project(e0, ngroups, nblk, 1, ctx->a_maxdeg, nullptr, P<EnvConst>(ctx->aw.envc), P<DevScene>(ctx->scene_table),
                   rp, ws, s);
    launch_tables_k(ec, ws.vcnt, ws.kcnt, P<uint64_t>(ctx->aw.kbase), P<uint32_t>(ctx->aw.blkbase), sort_block_size(),
                    ctx->a_kcap, ctx->a_nbcap, ok, err, s);
    ctx->launches += 5;
    TREC(2);
#ifdef GG_CHECK_PROTOCOLS
    CK(cudaMemsetAsync(ws.sorted, 0xff, ctx->a_kcap * 4, s));   // placement asserts each slot is written once
#endif
    ctx->launches += launch_sort_bin(ec, (uint32_t)ctx->a_nbcap, P<uint32_t>(ctx->aw.blkbase), P<uint32_t>(ctx->aw.blkenv),
                                     passes, rp, ws,
                                     P<uint32_t>(ctx->aw.ghist), P<uint32_t>(ctx->aw.thist), s, ctx->a_loop,
                                     P<uint32_t>(ctx->aw.qctr), tev ? tev[3] : nullptr);
    TREC(4);
    launch_raster(e0, ec, P<EnvConst>(ctx->aw.envc), rp, ws, rgb, depth, alpha, counters,
                  counters ? P<unsigned long long>(ctx->aw.counters) : nullptr, nullptr, -1, s);
    ctx->launches++;
    TREC(5);
    CK(cudaGetLastError());
  }
  if (ctx->timing) ctx->t_nchunks = nchunks;
  ctx->last_E = E;
  return GG_OK;
}

gg_status gg_reserve_async(gg_context* ctx, int32_t max_envs, int32_t W, int32_t H, int32_t chunk,
                           float max_visible_frac, float keys_per_visible) {
  if (!ctx) return GG_E_INVALID;
  const bool calibrated = max_visible_frac < 0.f;   // capacities from earlier synchronous renders
  if (max_envs <= 0 || W <= 0 || H <= 0 || chunk < 0 || !(max_visible_frac != 0.f) || max_visible_frac > 1.f ||
      (!calibrated && !(keys_per_visible > 0.f)) || !std::isfinite(max_visible_frac))
    return fail(ctx, GG_E_INVALID, "gg_reserve_async: bad arguments");
  if (calibrated && (ctx->cal_W != W || ctx->cal_H != H || ctx->cal_vmax == 0))
    return fail(ctx, GG_E_INVALID, "gg_reserve_async: calibrated capacities need a synchronous render at %dx%d first",
                W, H);
  if (ctx->scenes.empty()) return fail(ctx, GG_E_INVALID, "gg_reserve_async: load the scenes first");
  const int TX = (W + TILE - 1) / TILE, TY = (H + TILE - 1) / TILE, ntiles = TX * TY;
  if (ntiles > MAX_TILES) return fail(ctx, GG_E_UNSUPPORTED, "gg_reserve_async: image too large");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->own;
  // records per env the reservation provides for, then the chunk (the sync
  // workspace stays allocated, so only the async one counts as reusable)
  const double h = calibrated ? -(double)max_visible_frac : 0.0;
  const double rec_env = calibrated ? h * ctx->cal_vmean : (double)max_scene_n(ctx) * max_visible_frac;
  const int ch = chunk > 0 ? std::min(max_envs, chunk) : auto_chunk(ctx, max_envs, rec_env * 100.0, &ctx->aw);
  const int nmax = std::max(max_scene_n(ctx), 1);
  const int nblk = (nmax + PROJ_BLOCK - 1) / PROJ_BLOCK;
  int maxdeg = 0;
  for (const auto& sc : ctx->scenes)
    if (sc.live) maxdeg = std::max(maxdeg, sc.d.degree);
  uint64_t vcap, kcap;
  if (calibrated) {   // headroom h = -max_visible_frac over the densest observed chunk (and any single env)
    // small chunks vary most between pose sets: they get room for min(ch, 4)
    // envs at the largest single env seen; never more than every Gaussian
    const double few = (double)std::min(ch, 4);
    vcap = (uint64_t)std::min(h * std::max(ch * ctx->cal_vmean, few * ctx->cal_vmax), (double)ch * nmax) + 1;
    kcap = (uint64_t)(h * std::max(ch * ctx->cal_kmean, few * ctx->cal_kmax)) + 1;
  } else {
    vcap = (uint64_t)((double)ch * nmax * max_visible_frac) + 1;
    kcap = (uint64_t)((double)vcap * keys_per_visible) + 1;
  }
  const uint64_t nbcap = vcap / (uint64_t)sort_block_size() + ch + 1;
  bool okb = ensure(ctx, ctx->aw.envc, sizeof(EnvConst) * max_envs, s) && ensure(ctx, ctx->aw.perm, (size_t)max_envs * 4, s) &&
             ensure(ctx, ctx->aw.flags, (size_t)ch * nblk * PROJ_WPB * 4, s) && ensure(ctx, ctx->aw.blkcnt, (size_t)ch * nblk * 4, s) &&
             ensure(ctx, ctx->aw.vcnt, ch * 4, s) && ensure(ctx, ctx->aw.kcnt, ch * 8, s) && ensure(ctx, ctx->aw.rbase, ch * 8, s) &&
             ensure(ctx, ctx->aw.kbase, ch * 8, s) &&
             ensure(ctx, ctx->aw.ranges, (size_t)ch * ntiles * 8, s) && ensure(ctx, ctx->aw.okflag, 16, s) &&
             ensure(ctx, ctx->aw.counters, (size_t)max_envs * 32, s) && ensure(ctx, ctx->aw.rec0, vcap * 16, s) &&
             ensure(ctx, ctx->aw.rec1, vcap * 16, s) && ensure(ctx, ctx->aw.rec2, vcap * 16, s) &&
             ensure(ctx, ctx->aw.rect, vcap * 8, s) && ensure(ctx, ctx->aw.zkey, vcap * 4, s) &&
             ensure(ctx, ctx->aw.gid, vcap * 4, s) &&
             ensure(ctx, ctx->aw.rmask, vcap * 4 + 4, s) &&
             ensure(ctx, ctx->aw.dk0, vcap * 8, s) && ensure(ctx, ctx->aw.dk1, vcap * 8, s) &&
             ensure(ctx, ctx->aw.dv0, vcap * 4, s) &&
             ensure(ctx, ctx->aw.sorted, kcap * 4, s) && ensure(ctx, ctx->aw.blkbase, (size_t)(ch + 1) * 4, s) &&
             ensure(ctx, ctx->aw.blkenv, nbcap * 4 + 4, s) && ensure(ctx, ctx->aw.qctr, 64 * 4, s) &&
             ensure(ctx, ctx->aw.ghist, nbcap * sort_ghist_words() * 4, s) &&
             ensure(ctx, ctx->aw.thist, nbcap * ntiles * 4, s);
  CK(cudaStreamSynchronize(s));
  if (!okb) return fail(ctx, GG_E_OOM, "gg_reserve_async: allocation failed (%llu records, %llu keys)",
                        (unsigned long long)vcap, (unsigned long long)kcap);
  ctx->a_max_envs = max_envs; ctx->a_W = W; ctx->a_H = H; ctx->a_chunk = ch; ctx->a_nblk = nblk;
  ctx->a_maxdeg = maxdeg; ctx->a_vcap = vcap; ctx->a_kcap = kcap; ctx->a_nbcap = nbcap;
  // a calibrated capacity is within h of the blocks that exist, so the sync
  // kernels on a capacity-sized grid (surplus CTAs exit at once) beat the
  // bounded-grid work-counter variants (graph mode c3: depth stage 28.5 ->
  // 26.5 ms); a fraction-sized capacity may be far above them: keep the latter
  static const int env_loop = getenv("GG_ASYNC_LOOP") ? atoi(getenv("GG_ASYNC_LOOP")) : -1;   // A/B switch
  ctx->a_loop = env_loop >= 0 ? env_loop != 0 : !calibrated;
  ctx->async_ready = true;
  return GG_OK;
}

gg_status gg_render(gg_context* ctx, int32_t E, const int32_t* scene_ids, const float* viewmats,
                    const float* intr, int32_t W, int32_t H, const gg_render_opts* opts, void* rgb,
                    float* depth, float* alpha, void* stream) {
  if (!ctx) return GG_E_INVALID;
  if (opts && (opts->flags & GG_ASYNC)) {
    if (E <= 0 || !scene_ids || !viewmats || !intr || (opts->rgb_format != 0 && opts->rgb_format != 1) ||
        !(opts->near_plane > 0.f) || !(opts->far_plane > opts->near_plane) || opts->sh_degree > 3)
      return fail(ctx, GG_E_INVALID, "gg_render: bad arguments");
    CK(cudaSetDevice(ctx->device));
    return render_async(ctx, E, scene_ids, viewmats, intr, W, H, *opts, rgb, depth, alpha, (cudaStream_t)stream);
  }
  return render_impl(ctx, E, scene_ids, viewmats, intr, W, H, opts, rgb, depth, alpha,
                     (cudaStream_t)stream, nullptr, nullptr);
}

struct HostCopy {
  void* rgb_h; float* depth_h; float* alpha_h;
  uint8_t* rgb_d; float* depth_d; float* alpha_d;
  size_t rgb_px_bytes;
  int W, H;
  cudaStream_t s;
};

static gg_status copy_out_chunk(gg_context* ctx, int p0, int n, void* user) {
  HostCopy* h = (HostCopy*)user;
  const size_t P_ = (size_t)h->W * h->H;
  // the slice's outputs are final once its rasterisation completes: the copy
  // stream waits for that point and overlaps the copy with later work
  CK(cudaEventRecord(ctx->ev_copy, h->s));
  CK(cudaStreamWaitEvent(ctx->own, ctx->ev_copy, 0));
  // caller env indices of processing positions [p0, p0 + n), as sorted runs
  std::vector<int32_t> idx(ctx->h_perm + p0, ctx->h_perm + p0 + n);
  std::sort(idx.begin(), idx.end());
  for (size_t a = 0; a < idx.size();) {
    size_t b = a + 1;
    while (b < idx.size() && idx[b] == idx[b - 1] + 1) ++b;
    const size_t e0 = (size_t)idx[a], ec = b - a;
    if (h->rgb_h)
      CK(cudaMemcpyAsync((uint8_t*)h->rgb_h + e0 * P_ * h->rgb_px_bytes, h->rgb_d + e0 * P_ * h->rgb_px_bytes,
                         ec * P_ * h->rgb_px_bytes, cudaMemcpyDeviceToHost, ctx->own));
    if (h->depth_h)
      CK(cudaMemcpyAsync(h->depth_h + e0 * P_, h->depth_d + e0 * P_, ec * P_ * 4, cudaMemcpyDeviceToHost, ctx->own));
    if (h->alpha_h)
      CK(cudaMemcpyAsync(h->alpha_h + e0 * P_, h->alpha_d + e0 * P_, ec * P_ * 4, cudaMemcpyDeviceToHost, ctx->own));
    a = b;
  }
  return GG_OK;
}

// Host-buffer render.  Two device staging slots alternate between calls, so
// call t + 1 renders while call t's frames are still copying to the host: the
// render stream only waits (on the device) for the copies of call t - 1, which
// used the same slot.  The async form returns once everything is enqueued;
// gg_host_sync waits for every outstanding frame copy.
gg_status gg_render_host_async(gg_context* ctx, int32_t E, const int32_t* scene_ids, const float* viewmats,
                               const float* intr, int32_t W, int32_t H, const gg_render_opts* opts, void* rgb,
                               float* depth, float* alpha, void* stream) {
  if (!ctx) return GG_E_INVALID;
  if (E <= 0 || W <= 0 || H <= 0) return fail(ctx, GG_E_INVALID, "gg_render_host: bad sizes");
  if (!scene_ids || !viewmats || !intr) return fail(ctx, GG_E_INVALID, "gg_render_host: null input pointer");
  if (opts && (opts->flags & GG_ASYNC)) return fail(ctx, GG_E_UNSUPPORTED, "gg_render_host: GG_ASYNC needs device buffers");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int slot = ctx->h_slot;
  ctx->h_slot ^= 1;
  if (!ctx->h_done[slot]) CK(cudaEventCreateWithFlags(&ctx->h_done[slot], cudaEventDisableTiming));
  if (ctx->h_pending[slot]) CK(cudaStreamWaitEvent(s, ctx->h_done[slot], 0));   // slot's previous frames are out
  const int fmt = opts ? opts->rgb_format : 0;
  const size_t px = (size_t)W * H;
  const size_t rgb_px = fmt == 1 ? 12 : 3;
  const size_t in_bytes = (size_t)E * (4 + 64 + 16);
  const size_t out_rgb = rgb ? (size_t)E * px * rgb_px : 0;
  const size_t out_d = depth ? (size_t)E * px * 4 : 0;
  const size_t out_a = alpha ? (size_t)E * px * 4 : 0;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t total = al(in_bytes) + al(out_rgb) + al(out_d) + al(out_a);
  if (!ensure(ctx, ctx->h_in[slot], total, s)) return fail(ctx, GG_E_OOM, "gg_render_host: device staging");
  uint8_t* base = P<uint8_t>(ctx->h_in[slot]);
  int32_t* d_ids = (int32_t*)base;
  float* d_vm = (float*)(base + (size_t)E * 4);
  float* d_in = (float*)(base + (size_t)E * 68);
  uint8_t* d_rgb = base + al(in_bytes);
  float* d_depth = (float*)(base + al(in_bytes) + al(out_rgb));
  float* d_alpha = (float*)(base + al(in_bytes) + al(out_rgb) + al(out_d));
  CK(cudaMemcpyAsync(d_ids, scene_ids, (size_t)E * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_vm, viewmats, (size_t)E * 64, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_in, intr, (size_t)E * 16, cudaMemcpyHostToDevice, s));
  HostCopy hc{rgb, depth, alpha, d_rgb, d_depth, d_alpha, rgb_px, W, H, s};
  gg_status st = render_impl(ctx, E, d_ids, d_vm, d_in, W, H, opts, rgb ? (void*)d_rgb : nullptr,
                             depth ? d_depth : nullptr, alpha ? d_alpha : nullptr, s, copy_out_chunk, &hc);
  if (st != GG_OK) return st;
  CK(cudaEventRecord(ctx->h_done[slot], ctx->own));   // every frame copy of this call
  ctx->h_pending[slot] = true;
  return GG_OK;
}

gg_status gg_host_sync(gg_context* ctx) {
  if (!ctx) return GG_E_INVALID;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->own));
  ctx->h_pending[0] = ctx->h_pending[1] = false;
  return GG_OK;
}

gg_status gg_render_host(gg_context* ctx, int32_t E, const int32_t* scene_ids, const float* viewmats,
                         const float* intr, int32_t W, int32_t H, const gg_render_opts* opts, void* rgb,
                         float* depth, float* alpha, void* stream) {
  gg_status st = gg_render_host_async(ctx, E, scene_ids, viewmats, intr, W, H, opts, rgb, depth, alpha, stream);
  if (st != GG_OK) return st;
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return gg_host_sync(ctx);
}

gg_status gg_blur_poses(gg_context* ctx, int32_t E, const float* viewmats, const float* lin, const float* ang,
                        float shutter, int32_t K, float* out, void* stream) {
  if (!ctx) return GG_E_INVALID;
  if (E <= 0 || K < 1 || K > 64 || !(shutter >= 0.f) || !viewmats || !lin || !ang || !out)
    return fail(ctx, GG_E_INVALID, "gg_blur_poses: bad arguments");
  CK(cudaSetDevice(ctx->device));
  launch_blur_poses(E, K, K, viewmats, lin, ang, shutter, out, (cudaStream_t)stream);
  ctx->launches++;
  CK(cudaGetLastError());
  return GG_OK;
}

gg_status gg_render_blur(gg_context* ctx, int32_t E, const int32_t* scene_ids, const float* viewmats,
                         const float* intr, const float* lin, const float* ang, float shutter, int32_t K,
                         int32_t W, int32_t H, const gg_render_opts* opts_in, void* rgb, float* depth, float* alpha,
                         void* stream) {
  if (!ctx) return GG_E_INVALID;
  if (E <= 0 || W <= 0 || H <= 0 || K < 1 || K > 64 || !(shutter >= 0.f))
    return fail(ctx, GG_E_INVALID, "gg_render_blur: bad sizes, K or shutter");
  if (!scene_ids || !viewmats || !intr || !lin || !ang)
    return fail(ctx, GG_E_INVALID, "gg_render_blur: null input pointer");
  gg_render_opts opts;
  if (opts_in) opts = *opts_in; else gg_default_opts(&opts);
  if (opts.rgb_format != 0 && opts.rgb_format != 1) return fail(ctx, GG_E_INVALID, "gg_render_blur: rgb_format");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t npx = (size_t)W * H;
  // Kc cameras per env: the K colour samples, plus the nominal pose (t = 0)
  // for the depth when K is even (odd K: sample (K-1)/2 is at t = 0; R34)
  const bool need_depth = depth != nullptr;
  const int Kc = K + ((K % 2 == 0 && need_depth) ? 1 : 0);
  const int dk = (K % 2 == 1) ? (K - 1) / 2 : K;
  const int ecb = std::max(1, std::min(E, auto_chunk(ctx, E * Kc, sync_env_bytes(ctx), &ctx->sw) / Kc));
  const size_t nk = (size_t)ecb * Kc;
  if (!ensure(ctx, ctx->blur_vm, nk * 64, s) || !ensure(ctx, ctx->blur_ids, nk * 4, s) ||
      !ensure(ctx, ctx->blur_intr, nk * 16, s))
    return fail(ctx, GG_E_OOM, "gg_render_blur: sample cameras");
  gg_render_opts sub = opts;
  sub.flags = opts.flags & (GG_TIGHT_TILES | GG_ELLIPSE_TILES);   // tile-list variants apply per sample
  sub.debug_env = -1;
  const BlurSpec bs{K, Kc, dk};
  ctx->t_nchunks = 0;
  ctx->t_append = true;   // the stage times cover every sample chunk of this call
  const size_t rgb_px = opts.rgb_format == 1 ? 12 : 3;
  for (int e0 = 0; e0 < E; e0 += ecb) {
    const int ec = std::min(ecb, E - e0);
    launch_blur_poses(ec, K, Kc, viewmats + (size_t)e0 * 16, lin + (size_t)e0 * 3, ang + (size_t)e0 * 3, shutter,
                      P<float>(ctx->blur_vm), s);
    launch_blur_expand(ec, Kc, scene_ids + e0, intr + (size_t)e0 * 4, P<int32_t>(ctx->blur_ids),
                       P<float>(ctx->blur_intr), s);
    ctx->launches += 2;
    CK(cudaGetLastError());
    // the raster averages each env's samples in registers and writes its frame once (fused, R34)
    gg_status st = render_impl(ctx, ec * Kc, P<int32_t>(ctx->blur_ids), P<float>(ctx->blur_vm),
                               P<float>(ctx->blur_intr), W, H, &sub,
                               rgb ? (void*)((uint8_t*)rgb + (size_t)e0 * npx * rgb_px) : nullptr,
                               depth ? depth + (size_t)e0 * npx : nullptr, alpha ? alpha + (size_t)e0 * npx : nullptr,
                               s, nullptr, nullptr, &bs);
    if (st != GG_OK) {
      ctx->t_append = false;
      return st;
    }
  }
  ctx->t_append = false;
  return GG_OK;
}

gg_status gg_dino_input(gg_context* ctx, int32_t E, int32_t W, int32_t H, const uint8_t* rgb, int32_t S,
                        void* out, void* stream) {
  if (!ctx) return GG_E_INVALID;
  if (E <= 0 || W <= 0 || H <= 0 || S <= 0 || !rgb || !out)
    return fail(ctx, GG_E_INVALID, "gg_dino_input: bad arguments");
  CK(cudaSetDevice(ctx->device));
  launch_dino_input(E, W, H, S, rgb, out, (cudaStream_t)stream);
  ctx->launches++;
  CK(cudaGetLastError());
  return GG_OK;
}

gg_status gg_checksum(gg_context* ctx, int32_t E, int32_t W, int32_t H, const void* rgb, int32_t fmt,
                      const float* depth, uint64_t* out, void* stream) {
  if (!ctx) return GG_E_INVALID;
  if (E <= 0 || W <= 0 || H <= 0 || !out) return fail(ctx, GG_E_INVALID, "gg_checksum: bad args");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemsetAsync(out, 0, (size_t)E * 8, s));
  launch_checksum(E, W, H, fmt == 0 ? (const uint8_t*)rgb : nullptr, fmt == 1 ? (const float*)rgb : nullptr, depth,
                  (unsigned long long*)out, s);
  ctx->launches++;
  CK(cudaGetLastError());
  return GG_OK;
}

gg_status gg_check_errors(gg_context* ctx, void* stream) {
  if (!ctx) return GG_E_INVALID;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  CK(cudaMemcpy(ctx->h_err, ctx->errflag.p, 4, cudaMemcpyDeviceToHost));
  if (*ctx->h_err & ERR_BAD_SCENE) return fail(ctx, GG_E_BAD_SCENE, "device error: unknown scene id");
  if (*ctx->h_err & ERR_CAPACITY) return fail(ctx, GG_E_CAPACITY, "device error: capacity");
  return GG_OK;
}

gg_status gg_get_counters(gg_context* ctx, int32_t E, int64_t* dst) {
  if (!ctx || !dst || E <= 0) return GG_E_INVALID;
  const DevBuf* cb = ctx->last_counters;
  if (E > ctx->last_E || !cb || !cb->p || cb->bytes < (size_t)E * 32)
    return fail(ctx, GG_E_INVALID, "gg_get_counters: no counters for %d envs", E);
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(dst, cb->p, (size_t)E * 32, cudaMemcpyDeviceToHost));
  return GG_OK;
}

gg_status gg_debug_dump(gg_context* ctx, int32_t kind, void* dst, int64_t cap, int64_t* out_len) {
  if (!ctx || !out_len) return GG_E_INVALID;
  const void* src = nullptr;
  size_t n = 0, es = 4;
  switch (kind) {
    case GG_DUMP_TILE_COUNTS: src = ctx->d_tc.data(); n = ctx->d_tc.size(); break;
    case GG_DUMP_SORTED_TILE: src = ctx->d_stile.data(); n = ctx->d_stile.size(); break;
    case GG_DUMP_SORTED_ZBITS: src = ctx->d_sz.data(); n = ctx->d_sz.size(); break;
    case GG_DUMP_SORTED_GIDS: src = ctx->d_sgid.data(); n = ctx->d_sgid.size(); break;
    case GG_DUMP_RANGES: src = ctx->d_ranges.data(); n = ctx->d_ranges.size(); break;
    case GG_DUMP_COUNTERS: src = ctx->d_counters; n = 4; es = 8; break;
    case GG_DUMP_N_EVAL: src = ctx->d_neval.data(); n = ctx->d_neval.size(); break;
    case GG_DUMP_PROJ: src = ctx->d_proj.data(); n = ctx->d_proj.size(); break;
    default: return fail(ctx, GG_E_INVALID, "gg_debug_dump: unknown kind %d", kind);
  }
  *out_len = (int64_t)n;
  if (dst && cap > 0) memcpy(dst, src, std::min<size_t>(n, (size_t)cap) * es);
  return GG_OK;
}

}  // extern "C"
