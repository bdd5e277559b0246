// px_api.cu -- context, device memory and the C-ABI of libpx.so (include/px.h).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/px.h"
#include "px_kernels.h"

using namespace px;

namespace {

std::string g_create_error;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr, cap = 0;
    size_t want = bytes + bytes / 8 + 256;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr, cap = 0;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

struct ModelHost {
  int32_t object_id;
  int V, T;
  double cyl[3];
  DevBuf verts, col, tris;
};

struct CloudStore {  // ragged per-candidate clouds with capacity slots
  int64_t n = 0;
  long long total_cap = 0;
  bool organised = false;  // slot_map / bbox valid (rendered on the device)
  DevBuf bbox, cap, offset, count, points, lab, src, slot_map;
  void release() { bbox.release(), cap.release(), offset.release(), count.release(), points.release(), lab.release(), src.release(), slot_map.release(); }
};

}  // namespace

struct px_clouds {
  CloudStore s;
};

struct px_ctx {
  int device = 0;
  cudaStream_t stream = nullptr, own_stream = nullptr;
  std::string err;
  int64_t launches = 0;
  int64_t scratch_budget = (int64_t)8 << 30;
  // scene
  bool have_scene = false, organised = false;
  Camera cam{};
  int64_t n_obs = 0;
  DevBuf depth, valid, labels, obs_pts, obs_lab, obs_labels, obs_cell, gx, gy, gz, gidx;
  std::vector<int32_t> h_obs_labels, h_obs_src;
  bool obs_host_stale = false;  // the observed cloud was built on the device (px_scene_upload_frame): host copies lazily
  DevBuf obs_src, color_grid, row_cnt, row_off;
  DevBuf lat_objs, lat_rot, lat_tr;
  // models
  std::vector<ModelHost*> models;
  std::map<int32_t, int> slot_of;
  DevBuf models_dev, label_count;
  bool models_dirty = true;
  size_t render_smem = 0;
  // targets
  int n_targets = 0;
  long long tgt_total = 0;
  int tgt_k = 0;
  double tgt_gate = 0.0, tgt_eps = 0.0;
  DevBuf tgt_v0, tgt_obs, tgt_world, tgt_sizes, tgt_scans, tgt_params,
         tgt_off, tgt_pts, tgt_cov, tgt_soa, tgt_org, tgt_map, tgt_pix, tgt_boxes, tgt_lpts;
  bool tgt_organised = false;
  double tgt_rot[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};  // TargetsDev::rot of the resident targets
  bool tgt_obs_valid = false;  // tgt_obs holds the observed indices of the resident targets (device-built)
  // resident candidates
  int64_t n_cand = 0;
  bool have_tidx = false;
  DevBuf c_slot, c_pose, c_tidx, c_rank;
  // search scratch / results
  CloudStore clouds;
  DevBuf src_cov, w_buf, corr, nn, st_pose, st_i, st_hg, total_dev;
  long long refine_plane = 0;  // plane stride of the structure-of-arrays refine scratch
  DevBuf r_T, r_iters, r_flags, r_pose, r_jo, r_jr, r_nfirst, r_nfinal, r_key, bitmap, r_ncorr, r_cap0, r_cap1, r_nm, r_nfp;
  int bitmap_slots = 0;
  long long* total_host = nullptr;  // pinned
  void* frame_stage = nullptr;      // pinned staging of the stride-grid samples of a frame (px_scene_upload_frame_full)
  size_t frame_stage_cap = 0;
  double stage_ms[4] = {0, 0, 0, 0};
  bool kernel_timing = false;           // px_ctx_set_kernel_timing
  std::vector<cudaEvent_t> marks;       // per-launch event marks of the refine stage
  double kernel_ms[5] = {0, 0, 0, 0, 0};  // gicp init, nn, lin, halve, finish (last px_search_run)
  int64_t kernel_n[5] = {0, 0, 0, 0, 0};
  int chunks = 0;
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  // multi-GPU: this context's NCCL communicator (px_comm_init) and the per-object winner records
  void* comm = nullptr;
  int comm_rank = 0, comm_world = 1;
  DevBuf r_win, r_knife;
  bool win_valid = false;
  int32_t tidx_max = -1;  // largest resident target index (validated against n_targets at run time)
};

namespace {

int fail(px_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  else g_create_error = msg;
  return code;
}
#define CU(call)                                                                                      \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return fail(ctx, PX_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));                \
  } while (0)

int h2d(px_ctx* ctx, DevBuf& b, const void* src, size_t bytes) {
  CU(b.ensure(bytes ? bytes : 8));
  if (bytes) CU(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return 0;
}
int d2h(px_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes && dst) CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return 0;
}

int sync_models(px_ctx* ctx) {
  if (!ctx->models_dirty) return 0;
  std::vector<ModelDev> md(ctx->models.size());
  std::vector<int32_t> lc(ctx->models.size(), 0);
  size_t smem = 0;
  for (size_t i = 0; i < ctx->models.size(); ++i) {
    ModelHost* m = ctx->models[i];
    md[i].verts = m->verts.as<double>();
    md[i].col = m->col.as<double>();
    md[i].tris = m->tris.as<int32_t>();
    md[i].V = m->V, md[i].T = m->T, md[i].object_id = m->object_id, md[i].pad_ = 0;
    md[i].cyl_r2 = m->cyl[0], md[i].cyl_zmin = m->cyl[1], md[i].cyl_zmax = m->cyl[2];
    md[i].aabb_r = std::sqrt(m->cyl[0]) * (1.0 + 1e-9);
    smem = std::max(smem, render_smem_bytes(m->V, m->T));
    if (!ctx->obs_host_stale)
      for (int32_t l : ctx->h_obs_labels) lc[i] += (l == m->object_id);
  }
  ctx->render_smem = smem;
  if (int r = h2d(ctx, ctx->models_dev, md.data(), md.size() * sizeof(ModelDev))) return r;
  if (int r = h2d(ctx, ctx->label_count, lc.data(), lc.size() * sizeof(int32_t))) return r;
  if (ctx->obs_host_stale) {  // the labels of the observed cloud live on the device only
    CU(launch_label_count(ctx->obs_labels.as<int32_t>(), ctx->n_obs, ctx->models_dev.as<ModelDev>(), (int)md.size(),
                          ctx->label_count.as<int32_t>(), ctx->stream));
    ctx->launches += 1;
  }
  CU(cudaStreamSynchronize(ctx->stream));  // md / lc are stack-owned
  ctx->models_dirty = false;
  return 0;
}

int slots_from_ids(px_ctx* ctx, const int32_t* ids, int64_t n, std::vector<int32_t>& out) {
  out.resize((size_t)n);
  int32_t last_id = 0, last_slot = -1;  // candidates come in runs of one object
  for (int64_t i = 0; i < n; ++i) {
    if (last_slot < 0 || ids[i] != last_id) {
      auto it = ctx->slot_of.find(ids[i]);
      if (it == ctx->slot_of.end()) return fail(ctx, PX_E_ARG, "no model registered for id " + std::to_string(ids[i]));
      last_id = ids[i], last_slot = it->second;
    }
    out[(size_t)i] = last_slot;
  }
  return 0;
}

RenderArgs base_render_args(px_ctx* ctx) {
  RenderArgs a{};
  a.cam = ctx->cam;
  a.models = ctx->models_dev.as<ModelDev>();
  a.obs_depth = ctx->depth.as<double>();
  a.obs_valid = ctx->valid.as<uint8_t>();
  a.obs_labels = ctx->labels.as<int32_t>();
  return a;
}

// bbox + capacity scan for `n` candidates; returns total capacity via *total
int size_clouds(px_ctx* ctx, CloudStore& cs, const int32_t* slot_dev, const double* pose_dev, int64_t n,
                long long* total) {
  cs.n = n;
  CU(cs.bbox.ensure(sizeof(int4) * (size_t)n));
  CU(cs.cap.ensure(sizeof(long long) * (size_t)n));
  CU(cs.offset.ensure(sizeof(long long) * (size_t)n));
  CU(cs.count.ensure(sizeof(int32_t) * (size_t)n));
  RenderArgs a = base_render_args(ctx);
  a.model_slot = slot_dev, a.poses = pose_dev, a.n = (int)n;
  a.bbox = cs.bbox.as<int4>(), a.cap = cs.cap.as<long long>();
  CU(launch_bbox(a, ctx->stream));
  CU(launch_scan(cs.cap.as<long long>(), cs.offset.as<long long>(), ctx->total_dev.as<long long>(), (int)n, ctx->stream));
  ctx->launches += 2;
  CU(cudaMemcpyAsync(ctx->total_host, ctx->total_dev.p, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *total = *ctx->total_host;
  cs.total_cap = *total;
  return 0;
}

int render_clouds(px_ctx* ctx, CloudStore& cs, const int32_t* slot_dev, const double* pose_dev, int64_t n,
                  int occl, double delta_occ, int skip_lab = 0) {
  size_t tot = (size_t)std::max<long long>(cs.total_cap, 1);
  CU(cs.points.ensure(sizeof(double) * 3 * tot));
  CU(cs.lab.ensure(sizeof(double) * 3 * tot));
  CU(cs.src.ensure(sizeof(int32_t) * 2 * tot));
  CU(cs.slot_map.ensure(sizeof(int32_t) * tot));
  cs.organised = true;
  RenderArgs a = base_render_args(ctx);
  a.model_slot = slot_dev, a.poses = pose_dev, a.n = (int)n;
  a.occluder_marking = occl, a.delta_occ = delta_occ, a.skip_lab = skip_lab;
  a.bbox = cs.bbox.as<int4>(), a.cap = cs.cap.as<long long>(), a.offset = cs.offset.as<long long>();
  a.count = cs.count.as<int32_t>();
  a.points = cs.points.as<double>(), a.lab = cs.lab.as<double>(), a.src_px = cs.src.as<int32_t>();
  a.slot_map = cs.slot_map.as<int32_t>();
  CU(launch_render(a, ctx->render_smem, false, ctx->stream));
  ctx->launches += 1;
  return 0;
}

CloudsDev clouds_dev(const CloudStore& cs) {
  CloudsDev d{};
  d.n = (int)cs.n;
  d.offset = cs.offset.as<long long>();
  d.count = cs.count.as<int32_t>();
  d.points = cs.points.as<double>();
  d.lab = cs.lab.as<double>();
  d.src_px = cs.src.as<int32_t>();
  d.slot_map = cs.organised ? cs.slot_map.as<int32_t>() : nullptr;
  d.bbox = cs.organised ? cs.bbox.as<int4>() : nullptr;
  return d;
}

int ensure_bitmap(px_ctx* ctx) {
  const int words = (ctx->cam.GW * ctx->cam.GH + 31) / 32 + 1;
  const int slots = 148 * 32;  // one wave of persistent warps at 64 registers, whatever the CTA shape (multiple of PX_COST_WARPS)
  const size_t bytes = sizeof(uint32_t) * (size_t)words * slots;
  if (ctx->bitmap.cap < bytes || ctx->bitmap_slots != slots) {
    CU(ctx->bitmap.ensure(bytes));
    CU(cudaMemsetAsync(ctx->bitmap.p, 0, ctx->bitmap.cap, ctx->stream));
    ctx->bitmap_slots = slots;
  }
  return 0;
}

int run_cost(px_ctx* ctx, const CloudStore& cs, const int32_t* slot_dev, const double* cyl_pose_dev, double delta,
             double tau_c, int use_color, int32_t* jo_dev, int32_t* jr_dev, const int32_t* rank_dev,
             unsigned long long* key_dev, int lab_is_linear = 0, int32_t* nm_dev = nullptr, int32_t* nfp_dev = nullptr) {
  if (!ctx->organised) return fail(ctx, PX_E_ARG, "scene cloud is not the organised stride-grid cloud");
  if (int r = ensure_bitmap(ctx)) return r;
  CostArgs a{};
  a.ren = clouds_dev(cs);
  a.cam = ctx->cam;
  a.models = ctx->models_dev.as<ModelDev>();
  a.model_slot = slot_dev;
  a.cyl_poses = cyl_pose_dev;
  a.gx = ctx->gx.as<double>(), a.gy = ctx->gy.as<double>(), a.gz = ctx->gz.as<double>();
  a.gidx = ctx->gidx.as<int32_t>();
  a.obs_lab = ctx->obs_lab.as<double>();
  a.obs_labels = ctx->obs_labels.as<int32_t>();
  a.label_count = ctx->label_count.as<int32_t>();
  a.delta = delta, a.delta2 = delta * delta, a.tau_c = tau_c, a.use_color = use_color, a.lab_is_linear = lab_is_linear;
  a.bitmap = ctx->bitmap.as<uint32_t>();
  a.bitmap_words = (ctx->cam.GW * ctx->cam.GH + 31) / 32 + 1;
  a.bitmap_slots = ctx->bitmap_slots;
  a.j_o = jo_dev, a.j_r = jr_dev, a.rank = rank_dev, a.best_key = key_dev, a.n_match = nm_dev, a.n_foot = nfp_dev;
  a.knife = key_dev ? ctx->r_knife.as<unsigned long long>() : nullptr;  // fused search only
  CU(launch_cost(a, ctx->stream));
  ctx->launches += 1;
  return 0;
}

GicpCfgDev gicp_dev(const px_gicp_cfg& g) {
  GicpCfgDev d{};
  d.k_cov = g.k_covariance, d.max_iter = g.max_iterations, d.eps = g.epsilon;
  d.tol_t2 = g.translation_tolerance * g.translation_tolerance;
  d.tol_r2 = g.rotation_tolerance * g.rotation_tolerance;
  d.gate2 = g.max_correspondence_distance * g.max_correspondence_distance;
  return d;
}

int check_gicp(px_ctx* ctx, const px_gicp_cfg& g) {
  if (g.k_covariance < 4 || g.k_covariance > PX_KCOV_MAX)
    return fail(ctx, PX_E_LIMIT, "k_covariance must lie in [4, " + std::to_string(PX_KCOV_MAX) + "]");
  if (g.max_iterations < 0) return fail(ctx, PX_E_ARG, "max_iterations < 0");
  if (ctx->tgt_k != g.k_covariance || ctx->tgt_gate != g.max_correspondence_distance || ctx->tgt_eps != g.epsilon)
    return fail(ctx, PX_E_ARG, "targets were uploaded with a different k_covariance / epsilon / max_correspondence_distance");
  return 0;
}

int ensure_refine_scratch(px_ctx* ctx, long long total_cap, int64_t n_cand) {
  size_t tot = (size_t)std::max<long long>(total_cap, 1);
  CU(ctx->nn.ensure(sizeof(int32_t) * tot));
  CU(ctx->st_pose.ensure(sizeof(double) * 20 * (size_t)std::max<int64_t>(n_cand, 1)));
  CU(ctx->st_i.ensure(sizeof(int32_t) * 8 * (size_t)std::max<int64_t>(n_cand, 1)));
  CU(ctx->st_hg.ensure(sizeof(double) * 44 * (size_t)std::max<int64_t>(n_cand, 1)));
  ctx->refine_plane = (long long)tot;
  CU(ctx->src_cov.ensure(sizeof(double) * 6 * tot));  // x y z + covariance normal
  CU(ctx->w_buf.ensure(sizeof(double) * 10 * tot));
  return 0;
}

int set_camera(px_ctx* ctx, int32_t H, int32_t W, const double intr[4], int32_t stride) {
  if ((W + stride - 1) / stride > PX_TILE_PIX)
    return fail(ctx, PX_E_LIMIT, "image rows wider than " + std::to_string(PX_TILE_PIX) + " stride-grid pixels do not fit the z-buffer tile");
  Camera& c = ctx->cam;
  c.fx = intr[0], c.fy = intr[1], c.cx = intr[2], c.cy = intr[3];
  c.W = W, c.H = H, c.stride = stride;
  c.GW = (W + stride - 1) / stride, c.GH = (H + stride - 1) / stride;
  // bound of 1 + a^2 + b^2 over all pixel centres of the image (normalised coordinates)
  const double am = std::max(c.cx, (double)W - c.cx) / c.fx, bm = std::max(c.cy, (double)H - c.cy) / c.fy;
  c.ray_k = (double)stride / (std::max(c.fx, c.fy) * std::sqrt(1.0 + am * am + bm * bm)) * (1.0 - 1e-9);
  return 0;
}

// host copies of the observed labels / source pixels (needed by px_targets_upload's organised check only)
int fetch_obs_host(px_ctx* ctx) {
  if (!ctx->obs_host_stale) return 0;
  ctx->h_obs_labels.resize((size_t)ctx->n_obs);
  ctx->h_obs_src.resize(2 * (size_t)ctx->n_obs);
  if (int r = d2h(ctx, ctx->h_obs_labels.data(), ctx->obs_labels.p, (size_t)ctx->n_obs * 4)) return r;
  if (int r = d2h(ctx, ctx->h_obs_src.data(), ctx->obs_src.p, (size_t)ctx->n_obs * 8)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->obs_host_stale = false;
  return 0;
}

// ---- NCCL, bound at run time (no link-time dependency: torch ships libnccl.so.2) ----------------
struct px_nccl_id {
  char internal[128];  // ncclUniqueId (NCCL_UNIQUE_ID_BYTES)
};
struct NcclApi {
  void* handle = nullptr;
  int (*GetUniqueId)(px_nccl_id*) = nullptr;
  int (*CommInitRank)(void**, int, px_nccl_id, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*GetVersion)(int*) = nullptr;
} g_nccl;
enum { PX_NCCL_UINT64 = 5, PX_NCCL_MAX = 2, PX_NCCL_MIN = 3 };  // ncclDataType_t / ncclRedOp_t values (nccl.h)

int nccl_load(px_ctx* ctx, const char* path) {
  if (g_nccl.handle) return 0;
  void* h = nullptr;
  if (path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch already mapped
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(ctx, PX_E_ARG, std::string("cannot load NCCL: ") + dlerror());
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.GetVersion = (decltype(g_nccl.GetVersion))dlsym(h, "ncclGetVersion");
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.CommDestroy || !g_nccl.AllReduce || !g_nccl.GetErrorString)
    return fail(ctx, PX_E_ARG, "NCCL library lacks a required symbol");
  g_nccl.handle = h;
  return 0;
}
#define NC(call)                                                                                         \
  do {                                                                                                   \
    int r_ = (call);                                                                                     \
    if (r_ != 0) return fail(ctx, PX_E_CUDA, std::string(#call) + ": " + g_nccl.GetErrorString(r_));     \
  } while (0)

}  // namespace

// ---------------------------------------------------------------------------

extern "C" {

int px_ctx_create(int device, px_ctx** out) {
  px_ctx* ctx = nullptr;
  if (!out) return fail(nullptr, PX_E_ARG, "out is NULL");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, PX_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e) +
                                        " (libpx has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(nullptr, PX_E_ARG, "device index out of range");
  if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(nullptr, PX_E_CUDA, cudaGetErrorString(e));
  ctx = new px_ctx();
  ctx->device = device;
  if ((e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking)) != cudaSuccess) {
    delete ctx;
    return fail(nullptr, PX_E_CUDA, cudaGetErrorString(e));
  }
  ctx->stream = ctx->own_stream;
  cudaMallocHost((void**)&ctx->total_host, sizeof(long long));
  ctx->total_dev.ensure(sizeof(long long));
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  *out = ctx;
  return 0;
}

void px_ctx_destroy(px_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (ModelHost* m : ctx->models) {
    m->verts.release(), m->col.release(), m->tris.release();
    delete m;
  }
  DevBuf* bufs[] = {&ctx->depth, &ctx->valid, &ctx->labels, &ctx->obs_pts, &ctx->obs_lab, &ctx->obs_labels,
                    &ctx->gx, &ctx->gy, &ctx->gz, &ctx->gidx, &ctx->models_dev, &ctx->label_count,
                    &ctx->obs_cell, &ctx->tgt_v0, &ctx->tgt_obs, &ctx->tgt_world, &ctx->tgt_sizes, &ctx->tgt_scans, &ctx->tgt_params,
                    &ctx->tgt_off, &ctx->tgt_pts, &ctx->tgt_cov, &ctx->tgt_soa, &ctx->tgt_org, &ctx->tgt_map, &ctx->tgt_pix, &ctx->tgt_boxes, &ctx->tgt_lpts, &ctx->c_slot, &ctx->c_pose, &ctx->c_tidx,
                    &ctx->c_rank, &ctx->src_cov, &ctx->w_buf, &ctx->corr, &ctx->nn, &ctx->st_pose, &ctx->st_i, &ctx->st_hg, &ctx->total_dev, &ctx->r_T,
                    &ctx->r_iters, &ctx->r_flags, &ctx->r_pose, &ctx->r_jo, &ctx->r_jr, &ctx->r_nfirst,
                    &ctx->r_nfinal, &ctx->r_key, &ctx->bitmap, &ctx->r_ncorr, &ctx->r_cap0, &ctx->r_cap1, &ctx->r_nm, &ctx->r_nfp};
  for (DevBuf* b : bufs) b->release();
  ctx->r_win.release(), ctx->r_knife.release();
  ctx->obs_src.release(), ctx->color_grid.release(), ctx->row_cnt.release(), ctx->row_off.release();
  ctx->lat_objs.release(), ctx->lat_rot.release(), ctx->lat_tr.release();
  if (ctx->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(ctx->comm);
  ctx->comm = nullptr;
  ctx->clouds.release();
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t e : ctx->marks) cudaEventDestroy(e);
  if (ctx->total_host) cudaFreeHost(ctx->total_host);
  if (ctx->frame_stage) cudaFreeHost(ctx->frame_stage);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

const char* px_last_error(const px_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

int px_ctx_set_stream(px_ctx* ctx, void* s) {
  if (!ctx) return PX_E_ARG;
  cudaStreamSynchronize(ctx->stream);
  // NULL = the context's own non-blocking stream.  The legacy default stream has handle 0 as well, so it must be
  // named by CUDA's own sentinel cudaStreamLegacy ((void*)0x1); cudaStreamPerThread is (void*)0x2.
  ctx->stream = s ? (cudaStream_t)s : ctx->own_stream;
  return 0;
}

int px_ctx_sync(px_ctx* ctx) {
  if (!ctx) return PX_E_ARG;
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int px_ctx_set_scratch_budget(px_ctx* ctx, int64_t bytes) {
  if (!ctx || bytes < (1 << 20)) return fail(ctx, PX_E_ARG, "scratch budget too small");
  ctx->scratch_budget = bytes;
  return 0;
}

int64_t px_ctx_launch_count(const px_ctx* ctx) { return ctx ? ctx->launches : 0; }

int px_scene_upload(px_ctx* ctx, int32_t H, int32_t W, const double* depth, const uint8_t* valid,
                    const int32_t* labels, const double intr[4], int32_t stride, const double* obs_points,
                    const double* obs_lab, const int32_t* obs_src_px, const int32_t* obs_labels, int64_t n_obs) {
  if (!ctx) return PX_E_ARG;
  if (H <= 0 || W <= 0 || stride < 1 || !depth || !valid || !labels || !intr || n_obs < 0)
    return fail(ctx, PX_E_ARG, "px_scene_upload: bad arguments");
  CU(cudaSetDevice(ctx->device));
  if (int r = set_camera(ctx, H, W, intr, stride)) return r;
  Camera& c = ctx->cam;
  ctx->obs_host_stale = false;
  {
    // the batch path only ever reads the frame planes at the stride-grid pixels (raster.py:263-278): keep those
    const size_t ngrid = (size_t)c.GW * c.GH;
    std::vector<double> dg(ngrid);
    std::vector<uint8_t> vg(ngrid);
    std::vector<int32_t> lg(ngrid);
    for (int gv = 0; gv < c.GH; ++gv)
      for (int gu = 0; gu < c.GW; ++gu) {
        const size_t o = (size_t)gv * stride * W + (size_t)gu * stride, g = (size_t)gv * c.GW + gu;
        dg[g] = depth[o], vg[g] = valid[o], lg[g] = labels[o];
      }
    if (int r = h2d(ctx, ctx->depth, dg.data(), ngrid * sizeof(double))) return r;
    if (int r = h2d(ctx, ctx->valid, vg.data(), ngrid)) return r;
    if (int r = h2d(ctx, ctx->labels, lg.data(), ngrid * sizeof(int32_t))) return r;
    CU(cudaStreamSynchronize(ctx->stream));  // dg / vg / lg are stack-owned
  }
  if (int r = h2d(ctx, ctx->obs_pts, obs_points, (size_t)n_obs * 24)) return r;
  if (int r = h2d(ctx, ctx->obs_lab, obs_lab, (size_t)n_obs * 24)) return r;
  if (int r = h2d(ctx, ctx->obs_labels, obs_labels, (size_t)n_obs * 4)) return r;
  ctx->n_obs = n_obs;
  ctx->h_obs_labels.assign(obs_labels, obs_labels + n_obs);
  if (obs_src_px) ctx->h_obs_src.assign(obs_src_px, obs_src_px + 2 * n_obs);
  else ctx->h_obs_src.clear();
  // organised-grid view: valid iff every source pixel sits on the stride grid in
  // strictly increasing row-major order (what raster.frame_to_cloud produces)
  const size_t ng = (size_t)c.GW * c.GH;
  std::vector<double> gx(ng, NAN), gy(ng, NAN), gz(ng, NAN);
  std::vector<int32_t> gi(ng, -1);
  bool org = obs_src_px != nullptr;
  long long prev = -1;
  for (int64_t i = 0; org && i < n_obs; ++i) {
    const int u = obs_src_px[2 * i], v = obs_src_px[2 * i + 1];
    if (u < 0 || v < 0 || u >= W || v >= H || u % stride || v % stride) {
      org = false;
      break;
    }
    const long long g = (long long)(v / stride) * c.GW + u / stride;
    if (g <= prev) {
      org = false;
      break;
    }
    prev = g;
    gx[(size_t)g] = obs_points[3 * i], gy[(size_t)g] = obs_points[3 * i + 1], gz[(size_t)g] = obs_points[3 * i + 2];
    gi[(size_t)g] = (int32_t)i;
  }
  ctx->organised = org;
  std::vector<int32_t> cell((size_t)std::max<int64_t>(n_obs, 1), 0);
  if (org) {
    for (int64_t i = 0; i < n_obs; ++i)
      cell[(size_t)i] = (obs_src_px[2 * i + 1] / stride) * c.GW + obs_src_px[2 * i] / stride;
    if (int r = h2d(ctx, ctx->obs_cell, cell.data(), (size_t)n_obs * 4)) return r;
    if (int r = h2d(ctx, ctx->gx, gx.data(), ng * 8)) return r;
    if (int r = h2d(ctx, ctx->gy, gy.data(), ng * 8)) return r;
    if (int r = h2d(ctx, ctx->gz, gz.data(), ng * 8)) return r;
    if (int r = h2d(ctx, ctx->gidx, gi.data(), ng * 4)) return r;
  }
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->have_scene = true;
  ctx->models_dirty = true;  // label counts depend on the scene
  ctx->bitmap_slots = 0;     // grid size may have changed
  return 0;
}

int px_scene_upload_frame(px_ctx* ctx, int32_t H, int32_t W, const double* depth_grid, const uint8_t* valid_grid,
                          const int32_t* labels_grid, const double* color_grid, const double intr[4], int32_t stride,
                          int64_t* n_obs_out) {
  if (!ctx) return PX_E_ARG;
  if (H <= 0 || W <= 0 || stride < 1 || !depth_grid || !valid_grid || !labels_grid || !color_grid || !intr)
    return fail(ctx, PX_E_ARG, "px_scene_upload_frame: bad arguments");
  CU(cudaSetDevice(ctx->device));
  if (int r = set_camera(ctx, H, W, intr, stride)) return r;
  const Camera& c = ctx->cam;
  const size_t ng = (size_t)c.GW * c.GH;
  if (int r = h2d(ctx, ctx->depth, depth_grid, ng * sizeof(double))) return r;
  if (int r = h2d(ctx, ctx->valid, valid_grid, ng)) return r;
  if (int r = h2d(ctx, ctx->labels, labels_grid, ng * sizeof(int32_t))) return r;
  if (int r = h2d(ctx, ctx->color_grid, color_grid, ng * 24)) return r;
  CU(ctx->row_cnt.ensure((size_t)c.GH * 8));
  CU(ctx->row_off.ensure((size_t)c.GH * 8));
  SceneCloudArgs a{};
  a.H = H, a.W = W, a.stride = stride, a.GW = c.GW, a.GH = c.GH;
  a.fx = c.fx, a.fy = c.fy, a.cx = c.cx, a.cy = c.cy;
  a.depth = ctx->depth.as<double>(), a.valid = ctx->valid.as<uint8_t>(), a.labels = ctx->labels.as<int32_t>();
  a.color_grid = ctx->color_grid.as<double>();
  a.row_count = ctx->row_cnt.as<long long>(), a.row_offset = ctx->row_off.as<long long>();
  CU(launch_scene_count(a, ctx->stream));
  CU(launch_scan(a.row_count, ctx->row_off.as<long long>(), ctx->total_dev.as<long long>(), c.GH, ctx->stream));
  CU(cudaMemcpyAsync(ctx->total_host, ctx->total_dev.p, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  const int64_t n_obs = *ctx->total_host;
  const size_t n1 = (size_t)std::max<int64_t>(n_obs, 1);
  CU(ctx->obs_pts.ensure(n1 * 24));
  CU(ctx->obs_lab.ensure(n1 * 24));
  CU(ctx->obs_src.ensure(n1 * 8));
  CU(ctx->obs_labels.ensure(n1 * 4));
  CU(ctx->obs_cell.ensure(n1 * 4));
  CU(ctx->gx.ensure(ng * 8));
  CU(ctx->gy.ensure(ng * 8));
  CU(ctx->gz.ensure(ng * 8));
  CU(ctx->gidx.ensure(ng * 4));
  a.pts = ctx->obs_pts.as<double>(), a.lab = ctx->obs_lab.as<double>(), a.src = ctx->obs_src.as<int32_t>();
  a.labels_out = ctx->obs_labels.as<int32_t>(), a.cell = ctx->obs_cell.as<int32_t>();
  a.gx = ctx->gx.as<double>(), a.gy = ctx->gy.as<double>(), a.gz = ctx->gz.as<double>(), a.gidx = ctx->gidx.as<int32_t>();
  CU(launch_scene_fill(a, ctx->stream));
  ctx->launches += 3;
  ctx->n_obs = n_obs;
  ctx->organised = true, ctx->have_scene = true;
  ctx->obs_host_stale = true;
  ctx->h_obs_labels.clear(), ctx->h_obs_src.clear();
  ctx->models_dirty = true;
  ctx->bitmap_slots = 0;
  if (n_obs_out) *n_obs_out = n_obs;
  return 0;
}

int px_scene_upload_frame_full(px_ctx* ctx, int32_t H, int32_t W, const double* depth, const uint8_t* valid,
                               const int32_t* labels, const double* color, const double intr[4], int32_t stride,
                               int64_t* n_obs_out) {
  if (!ctx) return PX_E_ARG;
  if (H <= 0 || W <= 0 || stride < 1 || !depth || !valid || !labels || !color || !intr)
    return fail(ctx, PX_E_ARG, "px_scene_upload_frame_full: bad arguments");
  CU(cudaSetDevice(ctx->device));
  const int GW = (W + stride - 1) / stride, GH = (H + stride - 1) / stride;
  const size_t ng = (size_t)GW * GH;
  // one pinned block: depth (8 ng) | colour (24 ng) | labels (4 ng) | valid (ng)
  const size_t need = ng * 37 + 64;
  if (ctx->frame_stage_cap < need) {
    if (ctx->frame_stage) cudaFreeHost(ctx->frame_stage);
    ctx->frame_stage = nullptr, ctx->frame_stage_cap = 0;
    CU(cudaMallocHost(&ctx->frame_stage, need));
    ctx->frame_stage_cap = need;
  }
  CU(cudaStreamSynchronize(ctx->stream));  // a previous upload may still be reading the staging block
  double* sd = static_cast<double*>(ctx->frame_stage);
  double* sc = sd + ng;
  int32_t* sl = reinterpret_cast<int32_t*>(sc + 3 * ng);
  uint8_t* sv = reinterpret_cast<uint8_t*>(sl + ng);
  for (int gy = 0; gy < GH; ++gy) {
    const size_t row = (size_t)gy * stride * W;
    double* od = sd + (size_t)gy * GW;
    double* oc = sc + 3 * (size_t)gy * GW;
    int32_t* ol = sl + (size_t)gy * GW;
    uint8_t* ov = sv + (size_t)gy * GW;
    for (int gx = 0; gx < GW; ++gx) {
      const size_t px = row + (size_t)gx * stride;
      od[gx] = depth[px], ol[gx] = labels[px], ov[gx] = valid[px] ? 1 : 0;
      oc[3 * gx] = color[3 * px], oc[3 * gx + 1] = color[3 * px + 1], oc[3 * gx + 2] = color[3 * px + 2];
    }
  }
  return px_scene_upload_frame(ctx, H, W, sd, sv, sl, sc, intr, stride, n_obs_out);
}

int px_scene_download_cloud(px_ctx* ctx, double* points, double* lab, int32_t* src_px, int32_t* labels) {
  if (!ctx || !ctx->have_scene) return fail(ctx, PX_E_ARG, "px_scene_download_cloud: no scene");
  const size_t n = (size_t)ctx->n_obs;
  if (int r = d2h(ctx, points, ctx->obs_pts.p, n * 24)) return r;
  if (int r = d2h(ctx, lab, ctx->obs_lab.p, n * 24)) return r;
  if (labels)
    if (int r = d2h(ctx, labels, ctx->obs_labels.p, n * 4)) return r;
  if (src_px) {
    if (ctx->obs_host_stale || ctx->h_obs_src.empty()) {
      if (!ctx->obs_src.p) return fail(ctx, PX_E_ARG, "source pixels were not uploaded with this scene");
      if (int r = d2h(ctx, src_px, ctx->obs_src.p, n * 8)) return r;
    } else {
      memcpy(src_px, ctx->h_obs_src.data(), n * 8);
    }
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int px_model_upload(px_ctx* ctx, int32_t object_id, const double* verts, const double* colors_linear,
                    const int32_t* tris, int64_t V, int64_t T, const double cyl[3]) {
  if (!ctx) return PX_E_ARG;
  if (!verts || !colors_linear || V < 3 || T < 0 || (T && !tris) || !cyl)
    return fail(ctx, PX_E_ARG, "px_model_upload: bad arguments");
  if (T == 0) return fail(ctx, PX_E_ARG, "mesh has no triangles");
  for (int64_t i = 0; i < 3 * T; ++i)
    if (tris[i] < 0 || tris[i] >= V) return fail(ctx, PX_E_ARG, "triangle index out of range");
  if (render_smem_bytes((int)V, (int)T) > 220 * 1024)
    return fail(ctx, PX_E_LIMIT, "mesh too large for the shared-memory vertex cache (V <= ~7000)");
  CU(cudaSetDevice(ctx->device));
  ModelHost* m;
  auto it = ctx->slot_of.find(object_id);
  if (it == ctx->slot_of.end()) {
    m = new ModelHost();
    ctx->slot_of[object_id] = (int)ctx->models.size();
    ctx->models.push_back(m);
  } else {
    m = ctx->models[it->second];
  }
  m->object_id = object_id, m->V = (int)V, m->T = (int)T;
  m->cyl[0] = cyl[0], m->cyl[1] = cyl[1], m->cyl[2] = cyl[2];
  if (int r = h2d(ctx, m->verts, verts, (size_t)V * 24)) return r;
  if (int r = h2d(ctx, m->col, colors_linear, (size_t)V * 24)) return r;
  if (int r = h2d(ctx, m->tris, tris, (size_t)T * 12)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->models_dirty = true;
  return 0;
}

int px_model_count(const px_ctx* ctx) { return ctx ? (int)ctx->models.size() : 0; }
int px_model_ids(const px_ctx* ctx, int32_t* ids) {
  if (!ctx || !ids) return PX_E_ARG;
  for (size_t i = 0; i < ctx->models.size(); ++i) ids[i] = ctx->models[i]->object_id;
  return 0;
}

// ---- render_batch ----------------------------------------------------------

int px_render_batch(px_ctx* ctx, const int32_t* object_ids, const double* poses, int64_t n, int32_t occl,
                    double delta_occ, px_clouds** out) {
  if (!ctx || !out || n < 0 || (n && (!object_ids || !poses))) return fail(ctx, PX_E_ARG, "px_render_batch: bad arguments");
  if (!ctx->have_scene) return fail(ctx, PX_E_ARG, "no scene uploaded");
  if (n > 0x7fffffff) return fail(ctx, PX_E_LIMIT, "more than 2^31 candidates in one call");
  CU(cudaSetDevice(ctx->device));
  std::vector<int32_t> slots;
  if (int r = slots_from_ids(ctx, object_ids, n, slots)) return r;
  if (int r = sync_models(ctx)) return r;
  px_clouds* c = new px_clouds();
  DevBuf dslot, dpose;
  int rc = 0;
  do {
    if ((rc = h2d(ctx, dslot, slots.data(), (size_t)n * 4))) break;
    if ((rc = h2d(ctx, dpose, poses, (size_t)n * 96))) break;
    c->s.n = n;
    if (n) {
      long long total = 0;
      if ((rc = size_clouds(ctx, c->s, dslot.as<int32_t>(), dpose.as<double>(), n, &total))) break;
      if ((rc = render_clouds(ctx, c->s, dslot.as<int32_t>(), dpose.as<double>(), n, occl, delta_occ))) break;
    }
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, std::string("render: ") + cudaGetErrorString(e));
  } while (0);
  dslot.release(), dpose.release();
  if (rc) {
    c->s.release();
    delete c;
    return rc;
  }
  *out = c;
  return 0;
}

int64_t px_clouds_count(const px_clouds* c) { return c ? c->s.n : 0; }

int px_clouds_counts(px_ctx* ctx, const px_clouds* c, int32_t* counts) {
  if (!ctx || !c || !counts) return fail(ctx, PX_E_ARG, "px_clouds_counts: bad arguments");
  if (int r = d2h(ctx, counts, c->s.count.p, (size_t)c->s.n * 4)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int px_clouds_download(px_ctx* ctx, const px_clouds* c, double* points, double* lab, int32_t* src_px) {
  if (!ctx || !c) return fail(ctx, PX_E_ARG, "px_clouds_download: bad arguments");
  const int64_t n = c->s.n;
  if (n == 0) return 0;
  std::vector<int32_t> cnt((size_t)n);
  std::vector<long long> off((size_t)n);
  if (int r = d2h(ctx, cnt.data(), c->s.count.p, (size_t)n * 4)) return r;
  if (int r = d2h(ctx, off.data(), c->s.offset.p, (size_t)n * 8)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  // coalesce runs of candidates into few copies: slots are contiguous only when count == cap,
  // so stage the capacity-strided buffers on the host and compact there
  const size_t tot = (size_t)std::max<long long>(c->s.total_cap, 0);
  std::vector<double> hp, hl;
  std::vector<int32_t> hs;
  if (points) hp.resize(3 * tot);
  if (lab) hl.resize(3 * tot);
  if (src_px) hs.resize(2 * tot);
  if (int r = d2h(ctx, points ? hp.data() : nullptr, c->s.points.p, 24 * tot)) return r;
  if (int r = d2h(ctx, lab ? hl.data() : nullptr, c->s.lab.p, 24 * tot)) return r;
  if (int r = d2h(ctx, src_px ? hs.data() : nullptr, c->s.src.p, 8 * tot)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  size_t w = 0;
  for (int64_t i = 0; i < n; ++i) {
    const size_t k = (size_t)cnt[(size_t)i], o = (size_t)off[(size_t)i];
    if (points) memcpy(points + 3 * w, hp.data() + 3 * o, 24 * k);
    if (lab) memcpy(lab + 3 * w, hl.data() + 3 * o, 24 * k);
    if (src_px) memcpy(src_px + 2 * w, hs.data() + 2 * o, 8 * k);
    w += k;
  }
  return 0;
}

int px_clouds_upload(px_ctx* ctx, int64_t n, const int32_t* counts, const double* points, const double* lab,
                     const int32_t* src_px, px_clouds** out) {
  if (!ctx || !out || n < 0 || (n && !counts)) return fail(ctx, PX_E_ARG, "px_clouds_upload: bad arguments");
  CU(cudaSetDevice(ctx->device));
  std::vector<long long> off((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (counts[i] < 0) return fail(ctx, PX_E_ARG, "negative cloud size");
    off[(size_t)i + 1] = off[(size_t)i] + counts[i];
  }
  const size_t tot = (size_t)off[(size_t)n];
  if (tot && !points) return fail(ctx, PX_E_ARG, "points is NULL");
  px_clouds* c = new px_clouds();
  c->s.n = n, c->s.total_cap = (long long)tot;
  int rc = 0;
  do {
    if ((rc = h2d(ctx, c->s.offset, off.data(), (size_t)n * 8))) break;
    if ((rc = h2d(ctx, c->s.count, counts, (size_t)n * 4))) break;
    if ((rc = h2d(ctx, c->s.points, points, tot * 24))) break;
    std::vector<double> zl;
    std::vector<int32_t> zs;
    if (!lab) zl.assign(3 * tot + 1, 0.0);
    if (!src_px) zs.assign(2 * tot + 1, 0);
    if ((rc = h2d(ctx, c->s.lab, lab ? lab : zl.data(), tot * 24))) break;
    if ((rc = h2d(ctx, c->s.src, src_px ? src_px : zs.data(), tot * 8))) break;
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
  } while (0);
  if (rc) {
    c->s.release();
    delete c;
    return rc;
  }
  *out = c;
  return 0;
}

void px_clouds_free(px_ctx* ctx, px_clouds* c) {
  if (!c) return;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  c->s.release();
  delete c;
}

int px_rasterize(px_ctx* ctx, int32_t object_id, const double pose[12], double* zbuf, double* cbuf, uint8_t* valid,
                 int32_t* owner) {
  if (!ctx || !pose || !zbuf || !cbuf || !valid || !owner) return fail(ctx, PX_E_ARG, "px_rasterize: bad arguments");
  if (!ctx->have_scene) return fail(ctx, PX_E_ARG, "no scene uploaded (camera comes from the scene)");
  if (ctx->cam.W > PX_TILE_PIX)
    return fail(ctx, PX_E_LIMIT, "image rows wider than " + std::to_string(PX_TILE_PIX) + " pixels do not fit the z-buffer tile");
  CU(cudaSetDevice(ctx->device));
  std::vector<int32_t> slots;
  if (int r = slots_from_ids(ctx, &object_id, 1, slots)) return r;
  if (int r = sync_models(ctx)) return r;
  const size_t npix = (size_t)ctx->cam.W * ctx->cam.H;
  DevBuf dz, dc, dv, dow, dslot, dpose, dbb, dcap;
  int rc = 0;
  do {
    cudaError_t e;
    if ((e = dz.ensure(npix * 8)) || (e = dc.ensure(npix * 24)) || (e = dv.ensure(npix)) || (e = dow.ensure(npix * 4)) ||
        (e = dbb.ensure(sizeof(int4))) || (e = dcap.ensure(8))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    if ((rc = h2d(ctx, dslot, slots.data(), 4))) break;
    if ((rc = h2d(ctx, dpose, pose, 96))) break;
    RenderArgs a = base_render_args(ctx);
    a.cam.stride = 1, a.cam.GW = a.cam.W, a.cam.GH = a.cam.H;
    a.model_slot = dslot.as<int32_t>(), a.poses = dpose.as<double>(), a.n = 1;
    a.bbox = dbb.as<int4>(), a.cap = dcap.as<long long>();
    a.dense_z = dz.as<double>(), a.dense_c = dc.as<double>(), a.dense_valid = dv.as<uint8_t>(), a.dense_owner = dow.as<int32_t>();
    if ((e = launch_fill_dense(a.dense_z, a.dense_c, a.dense_valid, a.dense_owner, npix, ctx->stream)) ||
        (e = launch_bbox(a, ctx->stream)) || (e = launch_render(a, ctx->render_smem, true, ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    ctx->launches += 3;
    if ((rc = d2h(ctx, zbuf, dz.p, npix * 8)) || (rc = d2h(ctx, cbuf, dc.p, npix * 24)) ||
        (rc = d2h(ctx, valid, dv.p, npix)) || (rc = d2h(ctx, owner, dow.p, npix * 4)))
      break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, std::string("rasterize: ") + cudaGetErrorString(e));
  } while (0);
  DevBuf* bufs[] = {&dz, &dc, &dv, &dow, &dslot, &dpose, &dbb, &dcap};
  for (DevBuf* b : bufs) b->release();
  return rc;
}

// ---- registration -----------------------------------------------------------

int px_covariances(px_ctx* ctx, const double* points, int64_t n, int32_t k, double eps, double* cov_out) {
  if (!ctx || !points || !cov_out) return fail(ctx, PX_E_ARG, "px_covariances: bad arguments");
  if (k < 4 || k > PX_KCOV_MAX) return fail(ctx, PX_E_LIMIT, "k out of range [4,32]");
  if (n <= k) return fail(ctx, PX_E_ARG, "need more than k points");
  CU(cudaSetDevice(ctx->device));
  DevBuf dp, dc, doff;
  long long off[2] = {0, (long long)n};
  int rc = 0;
  do {
    if ((rc = h2d(ctx, dp, points, (size_t)n * 24))) break;
    if ((rc = h2d(ctx, doff, off, sizeof off))) break;
    cudaError_t e = dc.ensure((size_t)n * 72);
    if (e) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    CovArgs a{};
    a.n_clouds = 1, a.offset = doff.as<long long>(), a.points = dp.as<double>(), a.cov = dc.as<double>(), a.k = k, a.eps = eps;
    if ((e = launch_cov(a, n, ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    ctx->launches += 1;
    if ((rc = d2h(ctx, cov_out, dc.p, (size_t)n * 72))) break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, std::string("covariances: ") + cudaGetErrorString(e));
  } while (0);
  dp.release(), dc.release(), doff.release();
  return rc;
}

static TargetsDev targets_dev(px_ctx* ctx) {
  TargetsDev t{};
  t.n_targets = ctx->n_targets;
  t.offset = ctx->tgt_off.as<long long>();
  t.points = ctx->tgt_pts.as<double>();
  t.cov = ctx->tgt_cov.as<double>();
  t.org = ctx->tgt_organised ? ctx->tgt_org.as<TgtOrg>() : nullptr;
  t.tmap = ctx->tgt_map.as<int32_t>();
  t.boxes32 = ctx->tgt_boxes.as<float>();
  t.leaf32 = ctx->tgt_lpts.as<float4>();
  t.soa = ctx->tgt_soa.as<double>();
  t.plane = std::max<long long>(ctx->tgt_total, 1);
  t.f = 1.0 - ctx->tgt_eps;
  memcpy(t.rot, ctx->tgt_rot, sizeof t.rot);
  return t;
}

int px_targets_upload(px_ctx* ctx, int32_t n_targets, const int64_t* offsets, const double* points,
                      const int64_t* obs_index, const px_gicp_cfg* cfg) {
  if (!ctx || !cfg || n_targets < 0 || (n_targets && !offsets)) return fail(ctx, PX_E_ARG, "px_targets_upload: bad arguments");
  const int k = cfg->k_covariance;
  const double gate = cfg->max_correspondence_distance;
  if (k < 4 || k > PX_KCOV_MAX) return fail(ctx, PX_E_LIMIT, "k_covariance out of range [4,32]");
  if (!(gate > 0.0)) return fail(ctx, PX_E_ARG, "max_correspondence_distance must be positive");
  if (!(gate <= PX_GATE_MAX)) return fail(ctx, PX_E_LIMIT, "max_correspondence_distance above 1e3 m (fp32 pruning thresholds must stay finite)");
  CU(cudaSetDevice(ctx->device));
  const long long total = n_targets ? (long long)offsets[n_targets] : 0;
  for (int i = 0; i < n_targets; ++i)
    if (offsets[i + 1] < offsets[i] || offsets[i + 1] - offsets[i] > 0x7fffffff)
      return fail(ctx, PX_E_ARG, "target offsets must be non-decreasing");
  if (total && !points) return fail(ctx, PX_E_ARG, "target points is NULL");
  std::vector<long long> off((size_t)n_targets + 1, 0);
  for (int i = 0; i <= n_targets && n_targets; ++i) off[(size_t)i] = (long long)offsets[i];

  for (long long i = 0; i < 3 * total; ++i)
    if (!std::isfinite(points[i])) return fail(ctx, PX_E_ARG, "non-finite target point");

  // organised views: valid when every target is an index-ascending subset of the
  // uploaded scene's organised observed cloud
  if (obs_index != nullptr && ctx->have_scene && ctx->organised)
    if (int r = fetch_obs_host(ctx)) return r;
  bool org = obs_index != nullptr && ctx->have_scene && ctx->organised && !ctx->h_obs_src.empty();
  std::vector<TgtOrg> orgs((size_t)n_targets);
  std::vector<int32_t> tmap, tpix;
  std::vector<double> boxes;   // {lo xyz, hi xyz} per node, converted to fp32 centre/half-extent below
  std::vector<float> boxes32, leaf32;
  if (org) {
    const int st = ctx->cam.stride;
    tpix.resize((size_t)total);
    long long map_total = 0, box_total = 0;
    for (int t = 0; t < n_targets && org; ++t) {
      const long long a = off[(size_t)t], b = off[(size_t)t + 1];
      int x0 = 1 << 30, y0 = 1 << 30, x1 = -1, y1 = -1;
      long long prev = -1;
      for (long long i = a; i < b; ++i) {
        const long long oi = obs_index[i];
        if (oi <= prev || oi >= ctx->n_obs) {
          org = false;
          break;
        }
        prev = oi;
        const int gx = ctx->h_obs_src[2 * oi] / st, gy = ctx->h_obs_src[2 * oi + 1] / st;
        x0 = std::min(x0, gx), x1 = std::max(x1, gx), y0 = std::min(y0, gy), y1 = std::max(y1, gy);
      }
      TgtOrg& o = orgs[(size_t)t];
      if (b > a) o.gx0 = x0, o.gy0 = y0, o.w = x1 - x0 + 1, o.h = y1 - y0 + 1;
      else o.gx0 = o.gy0 = 0, o.w = 1, o.h = 1;
      o.bw = (o.w + PX_BLK - 1) / PX_BLK, o.bh = (o.h + PX_BLK - 1) / PX_BLK;
      o.sw = (o.bw + PX_BLK - 1) / PX_BLK, o.sh = (o.bh + PX_BLK - 1) / PX_BLK;
      o.map_off = map_total, o.box_off = box_total;
      map_total += (long long)o.w * o.h;
      box_total += (long long)o.bw * o.bh + (long long)o.sw * o.sh;
    }
    if (org) {
      tmap.assign((size_t)map_total, -1);
      boxes.resize((size_t)box_total * 6);
      for (long long q = 0; q < box_total; ++q)
        for (int d = 0; d < 3; ++d) boxes[(size_t)(6 * q + d)] = INFINITY, boxes[(size_t)(6 * q + 3 + d)] = -INFINITY;
      for (int t = 0; t < n_targets; ++t) {
        const TgtOrg& o = orgs[(size_t)t];
        const long long a = off[(size_t)t], b = off[(size_t)t + 1];
        double* bb = boxes.data() + 6 * o.box_off;
        double* sb = bb + 6 * (long long)o.bw * o.bh;
        for (long long i = a; i < b; ++i) {
          const long long oi = obs_index[i];
          const int x = ctx->h_obs_src[2 * oi] / st - o.gx0, y = ctx->h_obs_src[2 * oi + 1] / st - o.gy0;
          const int cell = y * o.w + x;
          tmap[(size_t)(o.map_off + cell)] = (int32_t)(i - a);
          tpix[(size_t)i] = cell;
          double* nb[2] = {bb + 6 * ((y / PX_BLK) * o.bw + x / PX_BLK),
                           sb + 6 * ((y / (PX_BLK * PX_BLK)) * o.sw + x / (PX_BLK * PX_BLK))};
          for (double* n6 : nb)
            for (int d = 0; d < 3; ++d) {
              const double v = points[3 * i + d];
              if (v < n6[d]) n6[d] = v;
              if (v > n6[3 + d]) n6[3 + d] = v;
            }
        }
      }
    }
  }
  if (org) {
    // fp32 pruning copies: lo rounded down / hi rounded up (the fp32 box contains the exact one), and the per-target
    // bound `err` on all fp32 rounding in the tests.  Device layout per target (TgtOrg::box_off counts nodes; 17 per
    // super-block): for every super-block six planes {lox, loy, loz, hix, hiy, hiz} x 16 block slots (row-major
    // inside the super-block, slots outside the map are empty boxes), then the super-blocks' own {lo, hi}; and one
    // leaf record per block slot: planes x[16], y[16], z[16] over the block's 4x4 map cells (PX_FAR32 = no point).
    auto conv = [](const double* b6, float* lo3, float* hi3, int stride) {
      for (int d = 0; d < 3; ++d) {
        const double lo = b6[d], hi = b6[3 + d];
        float lf = PX_FAR32, hf = -PX_FAR32;  // empty node: distance overflows to +inf and is always pruned
        if (lo <= hi) {
          lf = (float)lo, hf = (float)hi;
          if ((double)lf > lo) lf = std::nextafterf(lf, -INFINITY);
          if ((double)hf < hi) hf = std::nextafterf(hf, INFINITY);
        }
        lo3[d * stride] = lf, hi3[d * stride] = hf;
      }
    };
    long long node_total = 0;
    std::vector<long long> new_off((size_t)n_targets);
    for (int t = 0; t < n_targets; ++t) {
      new_off[(size_t)t] = node_total;
      const long long ns = (long long)orgs[(size_t)t].sw * orgs[(size_t)t].sh;
      node_total += 17 * ns + (ns & 1);  // even: keeps every target's planes 16-byte aligned
    }
    boxes32.assign((size_t)node_total * 6, 0.f);
    leaf32.assign((size_t)node_total * 48, PX_FAR32);
    const double empty6[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int t = 0; t < n_targets; ++t) {
      TgtOrg& o = orgs[(size_t)t];
      const double* bbd = boxes.data() + 6 * o.box_off;
      const double* sbd = bbd + 6 * (long long)o.bw * o.bh;
      float* out = boxes32.data() + 6 * new_off[(size_t)t];
      float* recs = leaf32.data() + 48 * new_off[(size_t)t];
      const int ns = o.sw * o.sh;
      for (int s_ = 0; s_ < ns; ++s_) {
        float* blk = out + 96 * (size_t)s_;
        for (int q = 0; q < 16; ++q) {
          const int by = (s_ / o.sw) * PX_BLK + (q >> 2), bx = (s_ % o.sw) * PX_BLK + (q & 3);
          const bool in = by < o.bh && bx < o.bw;
          conv(in ? bbd + 6 * ((long long)by * o.bw + bx) : empty6, blk + q, blk + 48 + q, 16);
        }
        float* sbo = out + 96 * (size_t)ns + 6 * (size_t)s_;
        conv(sbd + 6 * s_, sbo, sbo + 3, 1);
      }
      for (long long i = off[(size_t)t]; i < off[(size_t)t + 1]; ++i) {
        const int cell = tpix[(size_t)i], x = cell % o.w, y = cell / o.w;
        const int bx = x / PX_BLK, by = y / PX_BLK;
        const int s_ = (by / PX_BLK) * o.sw + bx / PX_BLK, q = (by % PX_BLK) * PX_BLK + bx % PX_BLK;
        float* rec = recs + 48 * ((size_t)16 * s_ + q);
        const int c = (y % PX_BLK) * PX_BLK + x % PX_BLK;
        for (int d = 0; d < 3; ++d) rec[16 * d + c] = (float)points[3 * i + d];
      }
      o.box_off = new_off[(size_t)t];
    }
    for (int t = 0; t < n_targets; ++t) {
      double m = 0.0;
      for (long long i = off[(size_t)t]; i < off[(size_t)t + 1]; ++i)
        for (int d = 0; d < 3; ++d) m = std::max(m, std::fabs(points[3 * i + d]));
      orgs[(size_t)t].err = std::ldexp(1.5 * (2.0 * m + gate + 1.0), -24);  // queries that can match: |q| <= m + gate
    }
  }
  ctx->tgt_organised = org, ctx->tgt_obs_valid = false;
  {
    const double I9[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};  // host-built structures are in the camera frame
    memcpy(ctx->tgt_rot, I9, sizeof I9);
  }

  if (int r = h2d(ctx, ctx->tgt_off, off.data(), off.size() * 8)) return r;
  if (int r = h2d(ctx, ctx->tgt_pts, points, (size_t)total * 24)) return r;
  if (org) {
    if (int r = h2d(ctx, ctx->tgt_org, orgs.data(), orgs.size() * sizeof(TgtOrg))) return r;
    if (int r = h2d(ctx, ctx->tgt_map, tmap.data(), tmap.size() * 4)) return r;
    if (int r = h2d(ctx, ctx->tgt_pix, tpix.data(), tpix.size() * 4)) return r;
    if (int r = h2d(ctx, ctx->tgt_boxes, boxes32.data(), boxes32.size() * 4)) return r;
    if (int r = h2d(ctx, ctx->tgt_lpts, leaf32.data(), leaf32.size() * 4)) return r;
  }
  const size_t tot1 = (size_t)std::max<long long>(total, 1);
  CU(ctx->tgt_cov.ensure(tot1 * 72));
  ctx->n_targets = n_targets, ctx->tgt_total = total, ctx->tgt_k = k, ctx->tgt_gate = gate, ctx->tgt_eps = cfg->epsilon;
  if (n_targets) {
    CovArgs a{};
    a.n_clouds = n_targets, a.offset = ctx->tgt_off.as<long long>(), a.count = nullptr;
    CU(ctx->tgt_v0.ensure(tot1 * 24));
    // targets of <= k points get no covariances (registration.py:504-510 skips them): zeros, not stale memory
    CU(cudaMemsetAsync(ctx->tgt_cov.p, 0, tot1 * 72, ctx->stream));
    CU(cudaMemsetAsync(ctx->tgt_v0.p, 0, tot1 * 24, ctx->stream));
    a.points = ctx->tgt_pts.as<double>(), a.cov = ctx->tgt_cov.as<double>(), a.v0 = ctx->tgt_v0.as<double>(), a.k = k, a.eps = cfg->epsilon;
    if (org) a.org = ctx->tgt_org.as<TgtOrg>(), a.tmap = ctx->tgt_map.as<int32_t>(), a.tpix = ctx->tgt_pix.as<int32_t>();
    a.ray_k = ctx->cam.ray_k;
    if (org) a.cam = ctx->cam;
    CU(launch_cov(a, total, ctx->stream));
    CU(ctx->tgt_soa.ensure(tot1 * 72));
    CU(launch_soa(ctx->tgt_pts.as<double>(), ctx->tgt_v0.as<double>(), ctx->tgt_soa.as<double>(), total, ctx->stream));
    ctx->launches += 2;
  }
  CU(cudaStreamSynchronize(ctx->stream));  // host staging vectors are stack-owned
  return 0;
}

// Common tail of the device-side target builders: sizes -> scans -> allocation -> fill -> covariances.
static int build_targets_device(px_ctx* ctx, TgtBuildArgs a, const px_gicp_cfg* cfg) {
  const int n = a.n_targets;
  const int k = cfg->k_covariance;
  if (k < 4 || k > PX_KCOV_MAX) return fail(ctx, PX_E_LIMIT, "k_covariance out of range [4,32]");
  if (!(cfg->max_correspondence_distance > 0.0)) return fail(ctx, PX_E_ARG, "max_correspondence_distance must be positive");
  if (!(cfg->max_correspondence_distance <= PX_GATE_MAX))
    return fail(ctx, PX_E_LIMIT, "max_correspondence_distance above 1e3 m (fp32 pruning thresholds must stay finite)");
  if (!ctx->have_scene || !ctx->organised) return fail(ctx, PX_E_ARG, "targets can only be cropped from an organised scene cloud");
  const size_t n1 = (size_t)std::max(n, 1);
  CU(ctx->tgt_sizes.ensure(3 * n1 * 8));
  CU(ctx->tgt_scans.ensure(2 * (n1 + 1) * 8));
  CU(ctx->tgt_off.ensure((n1 + 1) * 8));
  CU(ctx->tgt_org.ensure(n1 * sizeof(TgtOrg)));
  CU(ctx->tgt_world.ensure((size_t)std::max<int64_t>(ctx->n_obs, 1) * 24));
  a.obs_pts = ctx->obs_pts.as<double>(), a.obs_labels = ctx->obs_labels.as<int32_t>();
  a.obs_cell = ctx->obs_cell.as<int32_t>(), a.gidx = ctx->gidx.as<int32_t>(), a.n_obs = ctx->n_obs, a.GW = ctx->cam.GW;
  a.world = ctx->tgt_world.as<double>();
  a.gate = cfg->max_correspondence_distance;
  a.cam = ctx->cam;
  {
    // frame of the fp32 pruning structures: in 3-DoF the world frame, where the supporting plane (most of every
    // capsule crop) is axis-aligned; re-orthonormalised here (Gram-Schmidt in fp64) because the error bound of the
    // pruning tests assumes an isometry.  6-DoF label sub-clouds have no common plane: identity.
    double F[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    if (a.mode == 0 && n) {
      double r0[3] = {a.c2w[0], a.c2w[1], a.c2w[2]}, r1[3] = {a.c2w[4], a.c2w[5], a.c2w[6]};
      const double n0 = std::sqrt(r0[0] * r0[0] + r0[1] * r0[1] + r0[2] * r0[2]);
      for (double& v : r0) v /= n0;
      const double d01 = r0[0] * r1[0] + r0[1] * r1[1] + r0[2] * r1[2];
      for (int q = 0; q < 3; ++q) r1[q] -= d01 * r0[q];
      const double n1_ = std::sqrt(r1[0] * r1[0] + r1[1] * r1[1] + r1[2] * r1[2]);
      for (double& v : r1) v /= n1_;
      const double r2[3] = {r0[1] * r1[2] - r0[2] * r1[1], r0[2] * r1[0] - r0[0] * r1[2], r0[0] * r1[1] - r0[1] * r1[0]};
      if (std::isfinite(n0) && std::isfinite(n1_) && n0 > 0.5 && n1_ > 0.5)
        for (int q = 0; q < 3; ++q) F[q] = r0[q], F[3 + q] = r1[q], F[6 + q] = r2[q];
    }
    memcpy(a.frame, F, sizeof F);
    memcpy(ctx->tgt_rot, F, sizeof F);
  }
  a.cnt = ctx->tgt_sizes.as<long long>(), a.cells = a.cnt + n1, a.nodes = a.cells + n1;
  long long* off = ctx->tgt_off.as<long long>();
  long long* coff = ctx->tgt_scans.as<long long>();
  long long* noff = coff + n1 + 1;
  a.offset = off, a.cells_off = coff, a.nodes_off = noff;
  a.org = ctx->tgt_org.as<TgtOrg>();
  long long totals[3] = {0, 0, 0};
  if (n) {
    CU(launch_tgt_world(a, ctx->stream));
    CU(launch_tgt_count(a, ctx->stream));
    CU(launch_scan(a.cnt, off, off + n, n, ctx->stream));
    CU(launch_scan(a.cells, coff, coff + n, n, ctx->stream));
    CU(launch_scan(a.nodes, noff, noff + n, n, ctx->stream));
    ctx->launches += 5;
    CU(cudaMemcpyAsync(&totals[0], off + n, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(&totals[1], coff + n, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(&totals[2], noff + n, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  } else {
    CU(cudaMemsetAsync(off, 0, 8, ctx->stream));
  }
  const long long total = totals[0];
  const size_t tot1 = (size_t)std::max<long long>(total, 1);
  CU(ctx->tgt_obs.ensure(tot1 * 4));
  CU(ctx->tgt_pts.ensure(tot1 * 24));
  CU(ctx->tgt_pix.ensure(tot1 * 4));
  CU(ctx->tgt_map.ensure((size_t)std::max<long long>(totals[1], 1) * 4));
  CU(ctx->tgt_boxes.ensure((size_t)std::max<long long>(totals[2], 1) * 24));
  CU(ctx->tgt_lpts.ensure((size_t)std::max<long long>(totals[2], 1) * 192));
  CU(ctx->tgt_cov.ensure(tot1 * 72));
  CU(ctx->tgt_v0.ensure(tot1 * 24));
  CU(ctx->tgt_soa.ensure(tot1 * 72));
  a.tgt_obs = ctx->tgt_obs.as<int32_t>(), a.tgt_pts = ctx->tgt_pts.as<double>(), a.tpix = ctx->tgt_pix.as<int32_t>();
  a.tmap = ctx->tgt_map.as<int32_t>(), a.boxes32 = ctx->tgt_boxes.as<float>();
  a.leaf32 = ctx->tgt_lpts.as<float4>();
  ctx->tgt_organised = true, ctx->tgt_obs_valid = true;
  ctx->n_targets = n, ctx->tgt_total = total, ctx->tgt_k = k, ctx->tgt_gate = cfg->max_correspondence_distance;
  ctx->tgt_eps = cfg->epsilon;
  if (n) {
    CU(cudaMemsetAsync(a.tmap, 0xff, (size_t)std::max<long long>(totals[1], 1) * 4, ctx->stream));
    CU(launch_tgt_fill(a, ctx->stream));
    CovArgs c{};
    c.n_clouds = n, c.offset = off, c.count = nullptr;
    CU(cudaMemsetAsync(ctx->tgt_cov.p, 0, tot1 * 72, ctx->stream));  // targets of <= k points get none: zeros, not stale memory
    CU(cudaMemsetAsync(ctx->tgt_v0.p, 0, tot1 * 24, ctx->stream));
    c.points = a.tgt_pts, c.cov = ctx->tgt_cov.as<double>(), c.v0 = ctx->tgt_v0.as<double>(), c.k = k, c.eps = cfg->epsilon;
    c.org = a.org, c.tmap = a.tmap, c.tpix = a.tpix, c.ray_k = ctx->cam.ray_k, c.cam = ctx->cam;
    CU(launch_cov(c, total, ctx->stream));
    CU(launch_soa(a.tgt_pts, ctx->tgt_v0.as<double>(), ctx->tgt_soa.as<double>(), total, ctx->stream));
    ctx->launches += 5;
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int px_targets_build_capsules(px_ctx* ctx, int32_t n_targets, const double* params, const double cam_to_world[12],
                              const px_gicp_cfg* cfg) {
  if (!ctx || !cfg || n_targets < 0 || (n_targets && (!params || !cam_to_world)))
    return fail(ctx, PX_E_ARG, "px_targets_build_capsules: bad arguments");
  CU(cudaSetDevice(ctx->device));
  for (long long i = 0; i < 5LL * n_targets; ++i)
    if (!std::isfinite(params[i])) return fail(ctx, PX_E_ARG, "non-finite capsule parameter");
  if (int r = h2d(ctx, ctx->tgt_params, params, (size_t)n_targets * 40)) return r;
  TgtBuildArgs a{};
  a.n_targets = n_targets, a.mode = 0, a.params = ctx->tgt_params.as<double>();
  if (n_targets) memcpy(a.c2w, cam_to_world, sizeof a.c2w);
  return build_targets_device(ctx, a, cfg);
}

int px_targets_build_labels(px_ctx* ctx, int32_t n_targets, const int32_t* object_ids, const px_gicp_cfg* cfg) {
  if (!ctx || !cfg || n_targets < 0 || (n_targets && !object_ids))
    return fail(ctx, PX_E_ARG, "px_targets_build_labels: bad arguments");
  CU(cudaSetDevice(ctx->device));
  if (int r = h2d(ctx, ctx->tgt_params, object_ids, (size_t)n_targets * 4)) return r;
  TgtBuildArgs a{};
  a.n_targets = n_targets, a.mode = 1, a.label_ids = ctx->tgt_params.as<int32_t>();
  return build_targets_device(ctx, a, cfg);
}

int px_targets_info(px_ctx* ctx, int32_t* n_targets, int64_t* total_points) {
  if (!ctx) return PX_E_ARG;
  if (n_targets) *n_targets = ctx->n_targets;
  if (total_points) *total_points = ctx->tgt_total;
  return 0;
}

int px_targets_download(px_ctx* ctx, int64_t* offsets, double* points, int32_t* obs_index) {
  if (!ctx) return PX_E_ARG;
  CU(cudaSetDevice(ctx->device));
  if (int r = d2h(ctx, offsets, ctx->tgt_off.p, ((size_t)ctx->n_targets + 1) * 8)) return r;
  if (int r = d2h(ctx, points, ctx->tgt_pts.p, (size_t)ctx->tgt_total * 24)) return r;
  if (obs_index) {
    if (ctx->tgt_obs_valid) {
      if (int r = d2h(ctx, obs_index, ctx->tgt_obs.p, (size_t)ctx->tgt_total * 4)) return r;
    } else {
      for (long long i = 0; i < ctx->tgt_total; ++i) obs_index[i] = -1;  // uploaded targets carry no observed index
    }
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int px_targets_covariances(px_ctx* ctx, double* cov_out) {
  if (!ctx || !cov_out) return fail(ctx, PX_E_ARG, "px_targets_covariances: bad arguments");
  if (int r = d2h(ctx, cov_out, ctx->tgt_cov.p, (size_t)ctx->tgt_total * 72)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int px_refine_batch(px_ctx* ctx, const px_clouds* sources, const int32_t* target_idx, const double* init_T,
                    const px_gicp_cfg* cfg, double* out_T, int32_t* out_iters, int32_t* out_flags,
                    double* out_residual, double* out_trace, int32_t* out_ntrace) {
  if (!ctx || !sources || !cfg) return fail(ctx, PX_E_ARG, "px_refine_batch: bad arguments");
  const int64_t n = sources->s.n;
  if (n && !target_idx) return fail(ctx, PX_E_ARG, "target_idx is NULL");
  if (int r = check_gicp(ctx, *cfg)) return r;
  for (int64_t i = 0; i < n; ++i)
    if (target_idx[i] < 0 || target_idx[i] >= ctx->n_targets) return fail(ctx, PX_E_ARG, "target index out of range");
  if (n == 0) return 0;
  CU(cudaSetDevice(ctx->device));
  if (int r = ensure_refine_scratch(ctx, sources->s.total_cap, n)) return r;
  DevBuf dti, dinit, dT, dit, dfl, dres, dtr, dnt;
  int rc = 0;
  do {
    cudaError_t e;
    if ((rc = h2d(ctx, dti, target_idx, (size_t)n * 4))) break;
    if (init_T && (rc = h2d(ctx, dinit, init_T, (size_t)n * 96))) break;
    if ((e = dT.ensure((size_t)n * 96)) || (e = dit.ensure((size_t)n * 4)) || (e = dfl.ensure((size_t)n * 4)) ||
        (e = dnt.ensure((size_t)n * 4)) || (out_residual && (e = dres.ensure((size_t)n * 8))) ||
        (out_trace && (e = dtr.ensure((size_t)n * 16 * (size_t)std::max(cfg->max_iterations, 1))))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    // rows of the objective trace beyond a candidate's accepted steps are never written by the kernels: hand back zeros
    // (the reference's trace simply ends there), not whatever the allocation held
    if (out_trace && (e = cudaMemsetAsync(dtr.p, 0, (size_t)n * 16 * (size_t)std::max(cfg->max_iterations, 1), ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    RefineArgs a{};
    a.src = clouds_dev(sources->s);
    a.tgt = targets_dev(ctx);
    a.target_idx = dti.as<int32_t>();
    a.init_T = init_T ? dinit.as<double>() : nullptr;
    a.cfg = gicp_dev(*cfg);
    a.cam = ctx->cam;
    a.src_soa = ctx->src_cov.as<double>(), a.w_buf = ctx->w_buf.as<double>();
    a.plane = ctx->refine_plane;
    a.nn = ctx->nn.as<int32_t>(), a.st_pose = ctx->st_pose.as<double>(), a.st_i = ctx->st_i.as<int32_t>(), a.st_hg = ctx->st_hg.as<double>();
    a.out_T = dT.as<double>(), a.out_iters = dit.as<int32_t>(), a.out_flags = dfl.as<int32_t>();
    a.out_resid = out_residual ? dres.as<double>() : nullptr;
    a.out_trace = out_trace ? dtr.as<double>() : nullptr;
    a.out_ntrace = dnt.as<int32_t>();
    int nl = 0;
    if ((e = launch_refine(a, ctx->stream, &nl))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    ctx->launches += nl;
    if ((rc = d2h(ctx, out_T, dT.p, (size_t)n * 96)) || (rc = d2h(ctx, out_iters, dit.p, (size_t)n * 4)) ||
        (rc = d2h(ctx, out_flags, dfl.p, (size_t)n * 4)) || (rc = d2h(ctx, out_ntrace, dnt.p, (size_t)n * 4)) ||
        (out_residual && (rc = d2h(ctx, out_residual, dres.p, (size_t)n * 8))) ||
        (out_trace && (rc = d2h(ctx, out_trace, dtr.p, (size_t)n * 16 * (size_t)cfg->max_iterations))))
      break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, std::string("refine: ") + cudaGetErrorString(e));
  } while (0);
  DevBuf* bufs[] = {&dti, &dinit, &dT, &dit, &dfl, &dres, &dtr, &dnt};
  for (DevBuf* b : bufs) b->release();
  return rc;
}

// Test export: registration._gicp_linearize (registration.py:233-338) at the transform T for ONE source / target
// pair, through the production kernels (gicp_init_kernel covariances, gicp_nn_kernel, gicp_lin_kernel's ordered
// 43-lane sums).  Replaces the resident targets.
int px_gicp_linearize(px_ctx* ctx, const double* src, int64_t n, const double* tgt, int64_t m, const double T[12],
                      const px_gicp_cfg* cfg, double* h36, double* g6, double* f0, int32_t* n_corr, int64_t* corr,
                      double* w) {
  if (!ctx || !src || !tgt || !T || !cfg || n <= 0 || m <= 0) return fail(ctx, PX_E_ARG, "px_gicp_linearize: bad arguments");
  if (n <= cfg->k_covariance || m <= cfg->k_covariance) return fail(ctx, PX_E_ARG, "px_gicp_linearize: need more than k points");
  const int64_t offs[2] = {0, m};
  if (int r = px_targets_upload(ctx, 1, offs, tgt, nullptr, cfg)) return r;
  px_clouds* cl = nullptr;
  const int32_t cnt = (int32_t)n;
  if (int r = px_clouds_upload(ctx, 1, &cnt, src, nullptr, nullptr, &cl)) return r;
  int rc = 0;
  DevBuf dti, dinit, dT, dit, dfl;
  do {
    if ((rc = ensure_refine_scratch(ctx, cl->s.total_cap, 1))) break;
    const int32_t ti = 0;
    if ((rc = h2d(ctx, dti, &ti, 4)) || (rc = h2d(ctx, dinit, T, 96))) break;
    cudaError_t e;
    if ((e = dT.ensure(96)) || (e = dit.ensure(4)) || (e = dfl.ensure(4))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    RefineArgs a{};
    a.src = clouds_dev(cl->s);
    a.tgt = targets_dev(ctx);
    a.target_idx = dti.as<int32_t>(), a.init_T = dinit.as<double>();
    a.cfg = gicp_dev(*cfg);
    a.cfg.max_iter = std::max(a.cfg.max_iter, 1);
    a.cam = ctx->cam;
    a.src_soa = ctx->src_cov.as<double>(), a.w_buf = ctx->w_buf.as<double>(), a.plane = ctx->refine_plane;
    a.nn = ctx->nn.as<int32_t>(), a.st_pose = ctx->st_pose.as<double>(), a.st_i = ctx->st_i.as<int32_t>(), a.st_hg = ctx->st_hg.as<double>();
    a.out_T = dT.as<double>(), a.out_iters = dit.as<int32_t>(), a.out_flags = dfl.as<int32_t>();
    if ((e = launch_linearize_once(a, ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    ctx->launches += 3;
    double hg[44];
    int32_t sti[8];
    std::vector<int32_t> nn((size_t)n);
    const size_t plane = (size_t)ctx->refine_plane;
    std::vector<double> wb(10 * (size_t)n);
    if ((rc = d2h(ctx, hg, ctx->st_hg.p, sizeof hg)) || (rc = d2h(ctx, sti, ctx->st_i.p, sizeof sti)) ||
        (rc = d2h(ctx, nn.data(), ctx->nn.p, (size_t)n * 4)))
      break;
    for (int q = 0; q < 10 && !rc; ++q) rc = d2h(ctx, wb.data() + (size_t)q * n, ctx->w_buf.as<double>() + q * plane, (size_t)n * 8);
    if (rc) break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
      rc = fail(ctx, PX_E_CUDA, std::string("linearize: ") + cudaGetErrorString(e));
      break;
    }
    if (h36) memcpy(h36, hg, 36 * 8);
    if (g6) memcpy(g6, hg + 36, 6 * 8);
    if (f0) *f0 = hg[42];
    const int nc = sti[6];  // ST_NCOMPACT
    if (n_corr) *n_corr = nc;
    if (corr)
      for (int64_t i = 0; i < n; ++i) corr[i] = nn[(size_t)i];
    if (w) {
      memset(w, 0, (size_t)n * 72);
      for (int k = 0; k < nc; ++k) {
        long long ij;
        memcpy(&ij, &wb[9 * (size_t)n + k], 8);
        const size_t i = (size_t)(unsigned)ij;
        for (int q = 0; q < 9; ++q) w[9 * i + q] = wb[(size_t)q * n + k];
      }
    }
  } while (0);
  DevBuf* bufs[] = {&dti, &dinit, &dT, &dit, &dfl};
  for (DevBuf* b : bufs) b->release();
  px_clouds_free(ctx, cl);
  return rc;
}

// Test exports of the device colour functions (colorspace.py:41-124).
int px_ciede2000(px_ctx* ctx, const double* lab_a, const double* lab_b, int64_t n, double* out) {
  if (!ctx || n < 0 || (n && (!lab_a || !lab_b || !out))) return fail(ctx, PX_E_ARG, "px_ciede2000: bad arguments");
  if (n == 0) return 0;
  CU(cudaSetDevice(ctx->device));
  DevBuf da, db, dout;
  int rc = 0;
  do {
    if ((rc = h2d(ctx, da, lab_a, (size_t)n * 24)) || (rc = h2d(ctx, db, lab_b, (size_t)n * 24))) break;
    cudaError_t e;
    if ((e = dout.ensure((size_t)n * 8)) || (e = launch_ciede(da.as<double>(), db.as<double>(), dout.as<double>(), n, ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    ctx->launches += 1;
    if ((rc = d2h(ctx, out, dout.p, (size_t)n * 8))) break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
  } while (0);
  da.release(), db.release(), dout.release();
  return rc;
}

int px_srgb_to_lab(px_ctx* ctx, const double* rgb, int64_t n, int32_t linear_input, double* lab_out) {
  if (!ctx || n < 0 || (n && (!rgb || !lab_out))) return fail(ctx, PX_E_ARG, "px_srgb_to_lab: bad arguments");
  if (n == 0) return 0;
  CU(cudaSetDevice(ctx->device));
  DevBuf da, dout;
  int rc = 0;
  do {
    if ((rc = h2d(ctx, da, rgb, (size_t)n * 24))) break;
    cudaError_t e;
    if ((e = dout.ensure((size_t)n * 24)) || (e = launch_lab(da.as<double>(), dout.as<double>(), n, linear_input, ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    ctx->launches += 1;
    if ((rc = d2h(ctx, lab_out, dout.p, (size_t)n * 24))) break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
  } while (0);
  da.release(), dout.release();
  return rc;
}

// ---- cost ---------------------------------------------------------------------

int px_cost_batch(px_ctx* ctx, const px_clouds* rendered, const int32_t* object_ids, const double* cyl_poses,
                  double delta, double tau_c, int32_t use_color, int32_t* j_o, int32_t* j_r) {
  if (!ctx || !rendered || !j_o || !j_r) return fail(ctx, PX_E_ARG, "px_cost_batch: bad arguments");
  if (!ctx->have_scene) return fail(ctx, PX_E_ARG, "no scene uploaded");
  const int64_t n = rendered->s.n;
  if (n == 0) return 0;
  if (!object_ids) return fail(ctx, PX_E_ARG, "object_ids is NULL");
  CU(cudaSetDevice(ctx->device));
  std::vector<int32_t> slots;
  if (int r = slots_from_ids(ctx, object_ids, n, slots)) return r;
  if (int r = sync_models(ctx)) return r;
  DevBuf dslot, dpose, djo, djr;
  int rc = 0;
  do {
    cudaError_t e;
    if ((rc = h2d(ctx, dslot, slots.data(), (size_t)n * 4))) break;
    if (cyl_poses && (rc = h2d(ctx, dpose, cyl_poses, (size_t)n * 96))) break;
    if ((e = djo.ensure((size_t)n * 4)) || (e = djr.ensure((size_t)n * 4))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    if ((rc = run_cost(ctx, rendered->s, dslot.as<int32_t>(), cyl_poses ? dpose.as<double>() : nullptr, delta, tau_c,
                       use_color, djo.as<int32_t>(), djr.as<int32_t>(), nullptr, nullptr)))
      break;
    if ((rc = d2h(ctx, j_o, djo.p, (size_t)n * 4)) || (rc = d2h(ctx, j_r, djr.p, (size_t)n * 4))) break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, std::string("cost: ") + cudaGetErrorString(e));
  } while (0);
  dslot.release(), dpose.release(), djo.release(), djr.release();
  return rc;
}

int px_rendered_cost(px_ctx* ctx, const double* rp, const double* rlab, int64_t n_r, const double* op,
                     const double* olab, int64_t n_obs, double delta, double tau_c, int32_t use_color, int32_t* j_r,
                     uint8_t* explained) {
  if (!ctx || !j_r || n_r < 0 || n_obs < 0 || (n_obs && !explained)) return fail(ctx, PX_E_ARG, "px_rendered_cost: bad arguments");
  if (n_obs) memset(explained, 0, (size_t)n_obs);
  if (n_r == 0) {
    *j_r = 0;
    return 0;
  }
  if (n_obs == 0) {
    *j_r = (int32_t)n_r;
    return 0;
  }
  CU(cudaSetDevice(ctx->device));
  DevBuf drp, drl, dop, dol, dex, djr;
  int rc = 0;
  do {
    cudaError_t e;
    if ((rc = h2d(ctx, drp, rp, (size_t)n_r * 24)) || (rc = h2d(ctx, drl, rlab, (size_t)n_r * 24)) ||
        (rc = h2d(ctx, dop, op, (size_t)n_obs * 24)) || (rc = h2d(ctx, dol, olab, (size_t)n_obs * 24)))
      break;
    if ((e = dex.ensure((size_t)n_obs)) || (e = djr.ensure(4)) || (e = cudaMemsetAsync(dex.p, 0, (size_t)n_obs, ctx->stream)) ||
        (e = cudaMemsetAsync(djr.p, 0, 4, ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    GenericCostArgs a{drp.as<double>(), drl.as<double>(), (int)n_r, dop.as<double>(), dol.as<double>(), (long long)n_obs,
                      delta * delta, tau_c, use_color, dex.as<uint8_t>(), djr.as<int32_t>()};
    if ((e = launch_generic_cost(a, ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    ctx->launches += 1;
    if ((rc = d2h(ctx, j_r, djr.p, 4)) || (rc = d2h(ctx, explained, dex.p, (size_t)n_obs))) break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, std::string("rendered_cost: ") + cudaGetErrorString(e));
  } while (0);
  DevBuf* bufs[] = {&drp, &drl, &dop, &dol, &dex, &djr};
  for (DevBuf* b : bufs) b->release();
  return rc;
}

int px_knn(px_ctx* ctx, const double* q, int64_t nq, const double* t, int64_t nt, int32_t k, int64_t* idx, double* d2) {
  if (!ctx || nq < 0 || nt < 0 || k < 1 || (nq && (!q || !idx || !d2))) return fail(ctx, PX_E_ARG, "px_knn: bad arguments");
  if (k > PX_KCOV_MAX) return fail(ctx, PX_E_LIMIT, "k > 32");
  if (nq == 0) return 0;
  CU(cudaSetDevice(ctx->device));
  DevBuf dq, dt, di, dd;
  int rc = 0;
  do {
    cudaError_t e;
    if ((rc = h2d(ctx, dq, q, (size_t)nq * 24)) || (rc = h2d(ctx, dt, t, (size_t)nt * 24))) break;
    if ((e = di.ensure((size_t)nq * k * 8)) || (e = dd.ensure((size_t)nq * k * 8))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    KnnArgs a{dq.as<double>(), (long long)nq, dt.as<double>(), (long long)nt, k, di.as<long long>(), dd.as<double>()};
    if ((e = launch_knn(a, ctx->stream))) {
      rc = fail(ctx, PX_E_CUDA, cudaGetErrorString(e));
      break;
    }
    ctx->launches += 1;
    if ((rc = d2h(ctx, idx, di.p, (size_t)nq * k * 8)) || (rc = d2h(ctx, d2, dd.p, (size_t)nq * k * 8))) break;
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = fail(ctx, PX_E_CUDA, std::string("knn: ") + cudaGetErrorString(e));
  } while (0);
  dq.release(), dt.release(), di.release(), dd.release();
  return rc;
}

// ---- fused search -------------------------------------------------------------

int px_search_upload(px_ctx* ctx, int64_t n, const int32_t* object_ids, const double* poses, const int32_t* target_idx,
                     const int32_t* rank) {
  if (!ctx || n < 0 || (n && (!object_ids || !poses || !rank))) return fail(ctx, PX_E_ARG, "px_search_upload: bad arguments");
  if (n > 0x7fffffff) return fail(ctx, PX_E_LIMIT, "more than 2^31 candidates in one call");
  CU(cudaSetDevice(ctx->device));
  std::vector<int32_t> slots;
  if (int r = slots_from_ids(ctx, object_ids, n, slots)) return r;
  if (int r = h2d(ctx, ctx->c_slot, slots.data(), (size_t)n * 4)) return r;
  if (int r = h2d(ctx, ctx->c_pose, poses, (size_t)n * 96)) return r;
  if (int r = h2d(ctx, ctx->c_rank, rank, (size_t)n * 4)) return r;
  ctx->have_tidx = target_idx != nullptr;
  ctx->tidx_max = -1;
  if (target_idx) {
    for (int64_t i = 0; i < n; ++i) {
      if (target_idx[i] < 0) return fail(ctx, PX_E_ARG, "negative target index");
      ctx->tidx_max = std::max(ctx->tidx_max, target_idx[i]);
    }
    if (int r = h2d(ctx, ctx->c_tidx, target_idx, (size_t)n * 4)) return r;
  }
  CU(cudaStreamSynchronize(ctx->stream));  // `slots` is stack-owned
  ctx->n_cand = n;
  return 0;
}

int px_search_upload_lattice(px_ctx* ctx, int32_t mode3dof, int32_t n_objects, const px_lattice* objs,
                             const double world_to_cam[12], int32_t w2c_vec_order, const double cam_to_world[12],
                             const px_gicp_cfg* gicp, int32_t rank, int32_t world, int64_t* n_local_out) {
  if (!ctx || n_objects < 0 || (n_objects && !objs) || world < 1 || rank < 0 || rank >= world)
    return fail(ctx, PX_E_ARG, "px_search_upload_lattice: bad arguments");
  if (mode3dof && (!world_to_cam || (gicp && !cam_to_world))) return fail(ctx, PX_E_ARG, "px_search_upload_lattice: extrinsics missing");
  CU(cudaSetDevice(ctx->device));
  std::vector<LatticeObjDev> od((size_t)n_objects);
  std::vector<double> rot, tr;
  std::vector<int32_t> label_ids;
  long long n_local = 0;
  int n_targets = 0;
  for (int o = 0; o < n_objects; ++o) {
    const px_lattice& L = objs[o];
    if (L.n_outer <= 0 || L.n_inner <= 0 || !L.rotations || !L.translations)
      return fail(ctx, PX_E_ARG, "px_search_upload_lattice: empty lattice factor");
    auto it = ctx->slot_of.find(L.object_id);
    if (it == ctx->slot_of.end()) return fail(ctx, PX_E_ARG, "no model registered for id " + std::to_string(L.object_id));
    LatticeObjDev& d = od[(size_t)o];
    d.slot = it->second, d.n_outer = L.n_outer, d.n_inner = L.n_inner;
    d.n_outer_local = L.n_outer > rank ? (L.n_outer - rank + world - 1) / world : 0;
    d.cand_off = n_local;
    d.rot_off = (long long)rot.size() / 9, d.tr_off = (long long)tr.size() / 3;
    const int n_rot = mode3dof ? L.n_inner : L.n_outer, n_tr = mode3dof ? L.n_outer : L.n_inner;
    rot.insert(rot.end(), L.rotations, L.rotations + 9 * (size_t)n_rot);
    tr.insert(tr.end(), L.translations, L.translations + 3 * (size_t)n_tr);
    d.z_lo = L.capsule[0], d.z_hi = L.capsule[1], d.radius = L.capsule[2];
    d.tgt_off = n_targets, d.pad_ = 0;
    if (d.n_outer_local > 0) {  // objects without a local candidate get no target (plan order: first appearance)
      if (mode3dof) n_targets += d.n_outer_local;
      else n_targets += 1, label_ids.push_back(L.object_id);
    }
    n_local += (long long)d.n_outer_local * L.n_inner;
  }
  if (n_local > 0x7fffffff) return fail(ctx, PX_E_LIMIT, "more than 2^31 candidates in one call");
  const size_t n1 = (size_t)std::max<long long>(n_local, 1);
  if (int r = h2d(ctx, ctx->lat_objs, od.data(), od.size() * sizeof(LatticeObjDev))) return r;
  if (int r = h2d(ctx, ctx->lat_rot, rot.data(), rot.size() * 8)) return r;
  if (int r = h2d(ctx, ctx->lat_tr, tr.data(), tr.size() * 8)) return r;
  CU(ctx->c_slot.ensure(n1 * 4));
  CU(ctx->c_pose.ensure(n1 * 96));
  CU(ctx->c_rank.ensure(n1 * 4));
  CU(ctx->c_tidx.ensure(n1 * 4));
  const bool want_targets = gicp != nullptr;
  if (want_targets && mode3dof) CU(ctx->tgt_params.ensure((size_t)std::max(n_targets, 1) * 40));
  LatticeArgs a{};
  a.mode3dof = mode3dof, a.n_objects = n_objects, a.rank = rank, a.world = world, a.n_local = n_local;
  a.objs = ctx->lat_objs.as<LatticeObjDev>(), a.rotations = ctx->lat_rot.as<double>(), a.translations = ctx->lat_tr.as<double>();
  if (mode3dof) memcpy(a.w2c, world_to_cam, sizeof a.w2c);
  a.w2c_vec_order = w2c_vec_order;
  a.slot = ctx->c_slot.as<int32_t>(), a.poses = ctx->c_pose.as<double>(), a.rank_in_object = ctx->c_rank.as<int32_t>();
  a.tidx = want_targets ? ctx->c_tidx.as<int32_t>() : nullptr;
  a.capsules = want_targets && mode3dof ? ctx->tgt_params.as<double>() : nullptr;
  CU(launch_lattice(a, ctx->stream));
  if (n_local) ctx->launches += 1;
  CU(cudaStreamSynchronize(ctx->stream));  // od / rot / tr are stack-owned
  ctx->n_cand = n_local;
  ctx->have_tidx = want_targets;
  ctx->tidx_max = want_targets ? n_targets - 1 : -1;
  if (n_local_out) *n_local_out = n_local;
  if (!want_targets) return 0;
  if (mode3dof) {
    TgtBuildArgs t{};
    t.n_targets = n_targets, t.mode = 0, t.params = ctx->tgt_params.as<double>();
    memcpy(t.c2w, cam_to_world, sizeof t.c2w);
    return build_targets_device(ctx, t, gicp);
  }
  return px_targets_build_labels(ctx, (int32_t)label_ids.size(), label_ids.data(), gicp);
}

int px_search_candidates(px_ctx* ctx, int32_t* model_slot, double* poses, int32_t* target_idx, int32_t* rank_in_object) {
  if (!ctx) return PX_E_ARG;
  const size_t n = (size_t)ctx->n_cand;
  if (int r = d2h(ctx, model_slot, ctx->c_slot.p, n * 4)) return r;
  if (int r = d2h(ctx, poses, ctx->c_pose.p, n * 96)) return r;
  if (target_idx && ctx->have_tidx)
    if (int r = d2h(ctx, target_idx, ctx->c_tidx.p, n * 4)) return r;
  if (int r = d2h(ctx, rank_in_object, ctx->c_rank.p, n * 4)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

static int search_range(px_ctx* ctx, const px_search_cfg* cfg, int64_t lo, int64_t hi) {
  const bool timed = true;
  const int64_t n = hi - lo;
  if (n <= 0) return 0;
  const int32_t* slot = ctx->c_slot.as<int32_t>() + lo;
  const double* pose_in = ctx->c_pose.as<double>() + 12 * lo;
  double* pose_ref = ctx->r_pose.as<double>() + 12 * lo;
  long long total = 0;
  if (timed) CU(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (int r = size_clouds(ctx, ctx->clouds, slot, pose_in, n, &total)) return r;
  const long long per_slot = 60 + (cfg->refine ? 132 : 0);  // src planes 48, W + index planes 80, nn 4
  if (total * per_slot > ctx->scratch_budget && n > 1024) {
    const int64_t mid = lo + n / 2;
    if (int r = search_range(ctx, cfg, lo, mid)) return r;
    return search_range(ctx, cfg, mid, hi);
  }
  // with refinement on, the first render only feeds GICP (points); the colours are needed after the re-render
  if (int r = render_clouds(ctx, ctx->clouds, slot, pose_in, n, cfg->occluder_marking, cfg->delta, cfg->refine ? 1 : 2)) return r;
  CU(cudaMemcpyAsync(ctx->r_cap0.as<long long>() + lo, ctx->clouds.cap.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->r_nfirst.as<int32_t>() + lo, ctx->clouds.count.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  if (timed) CU(cudaEventRecord(ctx->ev[1], ctx->stream));
  const double* cost_pose = pose_in;
  size_t refine_marks = 0;
  if (cfg->refine) {
    if (int r = ensure_refine_scratch(ctx, total, n)) return r;
    RefineArgs a{};
    a.src = clouds_dev(ctx->clouds);
    a.tgt = targets_dev(ctx);
    a.target_idx = ctx->c_tidx.as<int32_t>() + lo;
    a.cfg = gicp_dev(cfg->gicp);
    a.cam = ctx->cam;
    a.src_soa = ctx->src_cov.as<double>(), a.w_buf = ctx->w_buf.as<double>();
    a.plane = ctx->refine_plane;
    a.nn = ctx->nn.as<int32_t>(), a.st_pose = ctx->st_pose.as<double>(), a.st_i = ctx->st_i.as<int32_t>(), a.st_hg = ctx->st_hg.as<double>();
    a.out_T = ctx->r_T.as<double>() + 12 * lo;
    a.out_iters = ctx->r_iters.as<int32_t>() + lo, a.out_flags = ctx->r_flags.as<int32_t>() + lo;
    a.out_ncorr_sum = ctx->r_ncorr.as<int32_t>() + lo;
    a.poses_in = pose_in, a.poses_out = pose_ref;
    a.mode3dof = cfg->mode3dof;
    memcpy(a.c2w, cfg->cam_to_world, sizeof a.c2w);
    memcpy(a.w2c, cfg->world_to_cam, sizeof a.w2c);
    a.c2w_vec_order = cfg->c2w_vec_order, a.w2c_vec_order = cfg->w2c_vec_order, a.fixed_z = cfg->fixed_z;
    int nl = 0;
    const size_t n_marks = ctx->kernel_timing ? 3 + 3 * (size_t)std::max(cfg->gicp.max_iterations, 0) : 0;
    while (ctx->marks.size() < n_marks) {
      cudaEvent_t e = nullptr;
      CU(cudaEventCreate(&e));
      ctx->marks.push_back(e);
    }
    CU(launch_refine(a, ctx->stream, &nl, n_marks ? ctx->marks.data() : nullptr));
    ctx->launches += nl;
    refine_marks = n_marks;
    if (timed) CU(cudaEventRecord(ctx->ev[2], ctx->stream));
    if (int r = size_clouds(ctx, ctx->clouds, slot, pose_ref, n, &total)) return r;
    if (int r = render_clouds(ctx, ctx->clouds, slot, pose_ref, n, cfg->occluder_marking, cfg->delta, 2)) return r;
    cost_pose = pose_ref;
  } else {
    CU(cudaMemcpyAsync(pose_ref, pose_in, (size_t)n * 96, cudaMemcpyDeviceToDevice, ctx->stream));
    if (timed) CU(cudaEventRecord(ctx->ev[2], ctx->stream));
  }
  CU(cudaMemcpyAsync(ctx->r_nfinal.as<int32_t>() + lo, ctx->clouds.count.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->r_cap1.as<long long>() + lo, ctx->clouds.cap.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  if (timed) CU(cudaEventRecord(ctx->ev[3], ctx->stream));
  if (int r = run_cost(ctx, ctx->clouds, slot, cfg->mode3dof ? cost_pose : nullptr, cfg->delta, cfg->tau_c, cfg->use_color,
                       ctx->r_jo.as<int32_t>() + lo, ctx->r_jr.as<int32_t>() + lo, ctx->c_rank.as<int32_t>() + lo,
                       ctx->r_key.as<unsigned long long>(), 1, ctx->r_nm.as<int32_t>() + lo, ctx->r_nfp.as<int32_t>() + lo))
    return r;
  if (timed) CU(cudaEventRecord(ctx->ev[4], ctx->stream));
  // per-chunk stage times accumulate (a split run is a sequence of such chunks)
  CU(cudaEventSynchronize(ctx->ev[4]));
  for (int i = 0; i < 4; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev[i], ctx->ev[i + 1]) == cudaSuccess) ctx->stage_ms[i] += ms;
  }
  for (size_t k = 0; k + 1 < refine_marks; ++k) {  // init, (nn, lin, halve) x iterations, finish
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->marks[k], ctx->marks[k + 1]) != cudaSuccess) continue;
    const int cls = k == 0 ? 0 : (k + 2 == refine_marks ? 4 : 1 + (int)((k - 1) % 3));
    ctx->kernel_ms[cls] += ms, ctx->kernel_n[cls] += 1;
  }
  ctx->chunks += 1;
  return 0;
}

int px_search_run(px_ctx* ctx, const px_search_cfg* cfg) {
  if (!ctx || !cfg) return fail(ctx, PX_E_ARG, "px_search_run: bad arguments");
  if (!ctx->have_scene) return fail(ctx, PX_E_ARG, "no scene uploaded");
  if (!ctx->organised) return fail(ctx, PX_E_ARG, "scene cloud is not the organised stride-grid cloud");
  CU(cudaSetDevice(ctx->device));
  const int64_t n = ctx->n_cand;
  if (cfg->refine) {
    if (!ctx->have_tidx) return fail(ctx, PX_E_ARG, "refine requested but no target_idx uploaded");
    if (int r = check_gicp(ctx, cfg->gicp)) return r;
    // the targets may have been replaced since px_search_upload (px_targets_*, px_refine_batch callers)
    if (ctx->tidx_max >= ctx->n_targets)
      return fail(ctx, PX_E_ARG, "resident candidates reference target " + std::to_string(ctx->tidx_max) + " but only " +
                                     std::to_string(ctx->n_targets) + " targets are resident");
  }
  if (int r = sync_models(ctx)) return r;
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  CU(ctx->r_T.ensure(nn * 96));
  CU(ctx->r_pose.ensure(nn * 96));
  DevBuf* ib[] = {&ctx->r_iters, &ctx->r_flags, &ctx->r_jo, &ctx->r_jr, &ctx->r_nfirst, &ctx->r_nfinal, &ctx->r_ncorr, &ctx->r_nm, &ctx->r_nfp};
  for (DevBuf* b : ib) CU(b->ensure(nn * 4));
  CU(ctx->r_cap0.ensure(nn * 8));
  CU(ctx->r_cap1.ensure(nn * 8));
  CU(cudaMemsetAsync(ctx->r_ncorr.p, 0, nn * 4, ctx->stream));
  CU(ctx->r_key.ensure(sizeof(unsigned long long) * std::max<size_t>(ctx->models.size(), 1)));
  CU(cudaMemsetAsync(ctx->r_key.p, 0xff, sizeof(unsigned long long) * std::max<size_t>(ctx->models.size(), 1), ctx->stream));
  CU(cudaMemsetAsync(ctx->r_iters.p, 0, nn * 4, ctx->stream));
  CU(cudaMemsetAsync(ctx->r_flags.p, 0, nn * 4, ctx->stream));
  {
    CU(ctx->r_knife.ensure(16));
    static const double inf2[2] = {INFINITY, INFINITY};
    CU(cudaMemcpyAsync(ctx->r_knife.p, inf2, 16, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (!cfg->refine) {
    // identity corrections
    std::vector<double> I((size_t)n * 12, 0.0);
    for (int64_t i = 0; i < n; ++i) I[12 * i] = I[12 * i + 5] = I[12 * i + 10] = 1.0;
    if (n) CU(cudaMemcpyAsync(ctx->r_T.p, I.data(), (size_t)n * 96, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  for (double& m : ctx->stage_ms) m = 0.0;
  for (int i = 0; i < 5; ++i) ctx->kernel_ms[i] = 0.0, ctx->kernel_n[i] = 0;
  ctx->win_valid = false;
  if (n == 0) return 0;
  ctx->chunks = 0;
  if (int r = search_range(ctx, cfg, 0, n)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int px_search_download(px_ctx* ctx, double* refined, double* reg_T, int32_t* iters, int32_t* flags, int32_t* j_o,
                       int32_t* j_r, int32_t* n_first, int32_t* n_final, uint64_t* best_key, double stage_ms[4]) {
  if (!ctx) return PX_E_ARG;
  const size_t n = (size_t)ctx->n_cand;
  if (int r = d2h(ctx, refined, ctx->r_pose.p, n * 96)) return r;
  if (int r = d2h(ctx, reg_T, ctx->r_T.p, n * 96)) return r;
  if (int r = d2h(ctx, iters, ctx->r_iters.p, n * 4)) return r;
  if (int r = d2h(ctx, flags, ctx->r_flags.p, n * 4)) return r;
  if (int r = d2h(ctx, j_o, ctx->r_jo.p, n * 4)) return r;
  if (int r = d2h(ctx, j_r, ctx->r_jr.p, n * 4)) return r;
  if (int r = d2h(ctx, n_first, ctx->r_nfirst.p, n * 4)) return r;
  if (int r = d2h(ctx, n_final, ctx->r_nfinal.p, n * 4)) return r;
  if (int r = d2h(ctx, best_key, ctx->r_key.p, ctx->models.size() * 8)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  if (stage_ms)
    for (int i = 0; i < 4; ++i) stage_ms[i] = ctx->stage_ms[i];
  return 0;
}

int px_ctx_set_kernel_timing(px_ctx* ctx, int32_t on) {
  if (!ctx) return PX_E_ARG;
  ctx->kernel_timing = on != 0;
  return 0;
}

int px_search_kernel_ms(px_ctx* ctx, double ms[5], int64_t launches[5]) {
  if (!ctx) return PX_E_ARG;
  for (int i = 0; i < 5; ++i) {
    if (ms) ms[i] = ctx->kernel_ms[i];
    if (launches) launches[i] = ctx->kernel_n[i];
  }
  return 0;
}

// ---- multi-GPU: the one collective ------------------------------------------------------------

int px_comm_unique_id(px_ctx* ctx, const char* nccl_path, uint8_t id[128]) {
  if (!id) return fail(ctx, PX_E_ARG, "px_comm_unique_id: id is NULL");
  if (int r = nccl_load(ctx, nccl_path)) return r;
  px_nccl_id u;
  NC(g_nccl.GetUniqueId(&u));
  memcpy(id, u.internal, sizeof u.internal);
  return 0;
}

int px_comm_init(px_ctx* ctx, const char* nccl_path, const uint8_t id[128], int32_t rank, int32_t world) {
  if (!ctx || !id || world < 1 || rank < 0 || rank >= world) return fail(ctx, PX_E_ARG, "px_comm_init: bad arguments");
  if (int r = nccl_load(ctx, nccl_path)) return r;
  CU(cudaSetDevice(ctx->device));
  if (ctx->comm) g_nccl.CommDestroy(ctx->comm), ctx->comm = nullptr;
  px_nccl_id u;
  memcpy(u.internal, id, sizeof u.internal);
  NC(g_nccl.CommInitRank(&ctx->comm, world, u, rank));
  ctx->comm_rank = rank, ctx->comm_world = world;
  return 0;
}

int px_comm_destroy(px_ctx* ctx) {
  if (!ctx) return PX_E_ARG;
  if (ctx->comm) {
    cudaStreamSynchronize(ctx->stream);
    g_nccl.CommDestroy(ctx->comm);
  }
  ctx->comm = nullptr, ctx->comm_rank = 0, ctx->comm_world = 1;
  return 0;
}

int px_comm_info(const px_ctx* ctx, int32_t* rank, int32_t* world, int32_t* nccl_version) {
  if (!ctx) return PX_E_ARG;
  if (rank) *rank = ctx->comm_rank;
  if (world) *world = ctx->comm ? ctx->comm_world : 1;
  if (nccl_version) {
    int v = 0;
    if (g_nccl.GetVersion) g_nccl.GetVersion(&v);
    *nccl_version = v;
  }
  return 0;
}

int px_search_reduce(px_ctx* ctx) {
  if (!ctx) return PX_E_ARG;
  CU(cudaSetDevice(ctx->device));
  const size_t nm = std::max<size_t>(ctx->models.size(), 1);
  unsigned long long* keys = ctx->r_key.as<unsigned long long>();
  if (!keys) return fail(ctx, PX_E_ARG, "px_search_reduce: no search has run");
  CU(ctx->r_win.ensure(nm * PX_WIN_WORDS * 8));
  unsigned long long* win = ctx->r_win.as<unsigned long long>();
  CU(cudaMemsetAsync(win, 0, nm * PX_WIN_WORDS * 8, ctx->stream));
  if (ctx->comm) NC(g_nccl.AllReduce(keys, keys, nm, PX_NCCL_UINT64, PX_NCCL_MIN, ctx->comm, ctx->stream));
  WinnerArgs a{};
  a.n = (int)ctx->n_cand;
  a.model_slot = ctx->c_slot.as<int32_t>(), a.rank = ctx->c_rank.as<int32_t>();
  a.j_o = ctx->r_jo.as<int32_t>(), a.j_r = ctx->r_jr.as<int32_t>(), a.n_final = ctx->r_nfinal.as<int32_t>();
  a.refined = ctx->r_pose.as<double>(), a.reg_T = ctx->r_T.as<double>();
  a.best_key = keys, a.win = win;
  CU(launch_winners(a, ctx->stream));
  if (a.n) ctx->launches += 1;
  if (ctx->comm) NC(g_nccl.AllReduce(win, win, nm * PX_WIN_WORDS, PX_NCCL_UINT64, PX_NCCL_MAX, ctx->comm, ctx->stream));
  ctx->win_valid = true;
  return 0;
}

int px_search_winners(px_ctx* ctx, uint64_t* best_key, double* refined, double* reg_T, int32_t* j_o, int32_t* j_r,
                      int32_t* max_points) {
  if (!ctx) return PX_E_ARG;
  if (!ctx->win_valid) return fail(ctx, PX_E_ARG, "px_search_winners: call px_search_reduce after px_search_run first");
  const size_t nm = ctx->models.size();
  std::vector<unsigned long long> w(std::max<size_t>(nm, 1) * PX_WIN_WORDS);
  if (int r = d2h(ctx, w.data(), ctx->r_win.p, w.size() * 8)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  for (size_t s = 0; s < nm; ++s) {
    const unsigned long long* r = w.data() + s * PX_WIN_WORDS;
    if (best_key) best_key[s] = r[0] ? r[0] - 1ull : UINT64_MAX;  // word 0 holds key + 1; 0 = no candidate anywhere
    for (int q = 0; q < 12; ++q) {
      if (refined) memcpy(&refined[12 * s + q], &r[1 + q], 8);
      if (reg_T) memcpy(&reg_T[12 * s + q], &r[13 + q], 8);
    }
    if (j_o) j_o[s] = (int32_t)r[25];
    if (j_r) j_r[s] = (int32_t)r[26];
    if (max_points) max_points[s] = (int32_t)r[27];
  }
  return 0;
}

int px_search_knife_edges(px_ctx* ctx, double margins[2]) {
  if (!ctx || !margins) return PX_E_ARG;
  if (!ctx->r_knife.p) return fail(ctx, PX_E_ARG, "px_search_knife_edges: no search has run");
  if (int r = d2h(ctx, margins, ctx->r_knife.p, 16)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int px_search_stats(px_ctx* ctx, int32_t* ncorr_sum, int64_t* cap_first, int64_t* cap_final, int32_t* n_match,
                    int32_t* n_footprint) {
  if (!ctx) return PX_E_ARG;
  const size_t n = (size_t)ctx->n_cand;
  if (int r = d2h(ctx, ncorr_sum, ctx->r_ncorr.p, n * 4)) return r;
  if (int r = d2h(ctx, n_match, ctx->r_nm.p, n * 4)) return r;
  if (int r = d2h(ctx, n_footprint, ctx->r_nfp.p, n * 4)) return r;
  if (int r = d2h(ctx, cap_first, ctx->r_cap0.p, n * 8)) return r;
  if (int r = d2h(ctx, cap_final, ctx->r_cap1.p, n * 8)) return r;
  CU(cudaStreamSynchronize(ctx->stream));
  return 0;
}

}  // extern "C"
