/*
 * px.h -- C-ABI of libpx.so, the B200 (sm_100a) implementation of the PERCH 2.0
 * parallel-search hot path: render -> GICP refine -> re-render -> cost -> argmin.
 *
 * The reference (Python package `rvpose`) has no FFI layer; its boundary for this
 * path is the Python API re-exported in pkg/src/rvpose/__init__.py:9-66.  Each
 * entry point below names the reference function it replaces (paths relative to
 * /root/reference/pkg/src/rvpose/).  INTEGRATION.md shows the ctypes binding a
 * maintainer of the reference would add.
 *
 * Conventions: plain pointers and sizes only; every array is C-contiguous;
 * float64 / int32 / uint8 as stated; the caller owns all host buffers, the
 * context owns all device memory; one context per device, not thread-safe; every
 * call is synchronous at return (inputs consumed, outputs written) unless noted.
 * Return value 0 = success, negative = error (PX_E_*); the message is available
 * from px_last_error().  There is no CPU fallback: without a CUDA device
 * px_ctx_create fails.
 */
#ifndef PX_H_
#define PX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PX_E_CUDA (-1)      /* CUDA runtime error */
#define PX_E_ARG (-2)       /* bad argument / unknown object id / state missing */
#define PX_E_LIMIT (-3)     /* implementation limit exceeded (see message) */

/* failure codes in the low byte of `flags` (registration.py:434-456, 504-510);
 * bit 8 (0x100) = converged */
#define PX_FAIL_NONE 0
#define PX_FAIL_TOO_FEW_POINTS 1
#define PX_FAIL_DEGENERATE_CORRESPONDENCES 2
#define PX_FAIL_SINGULAR_NORMAL_EQUATIONS 3
#define PX_FAIL_NO_DECREASE 4
#define PX_FLAG_CONVERGED 0x100

typedef struct px_ctx px_ctx;
typedef struct px_clouds px_clouds; /* device-resident ragged batch of LabeledCloud (model.py:185-217) */

/* GicpConfig, registration.py:26-42 */
typedef struct {
  int32_t k_covariance;                /* 4 .. 32, else PX_E_LIMIT */
  int32_t max_iterations;
  double epsilon;
  double translation_tolerance;
  double rotation_tolerance;
  double max_correspondence_distance;  /* metres, (0, 1000]: larger gates are refused with PX_E_LIMIT */
} px_gicp_cfg;

/* The part of SearchConfig (search.py:37-61) the per-candidate stages read, plus
 * the camera extrinsics used by the 3-DoF re-lift (search.py:295-299). */
typedef struct {
  int32_t mode3dof;          /* 1 = "3dof" (cylinder association, planar re-lift), 0 = "6dof" (labels) */
  int32_t use_color;
  int32_t occluder_marking;
  int32_t refine;
  double delta;              /* also delta_occ, search.py:276 */
  double tau_c;
  px_gicp_cfg gicp;
  double cam_to_world[12];   /* row-major 3x4 */
  double world_to_cam[12];
  int32_t c2w_vec_order;     /* 0: host rotation array is C-contiguous, 1: transposed view */
  int32_t w2c_vec_order;     /*    (selects numpy's (3,3)@(3,) rounding order) */
  double fixed_z;
} px_search_cfg;

/* ---- context ---------------------------------------------------------------- */
int px_ctx_create(int device, px_ctx** out);
void px_ctx_destroy(px_ctx* ctx);
const char* px_last_error(const px_ctx* ctx); /* ctx may be NULL: last creation error */
/* Launch on a caller-provided cudaStream_t (e.g. torch's current stream); NULL
 * restores the context's own (non-blocking) stream.  The legacy default stream
 * also has handle 0: name it by CUDA's sentinel cudaStreamLegacy, (void*)0x1. */
int px_ctx_set_stream(px_ctx* ctx, void* cuda_stream);
int px_ctx_sync(px_ctx* ctx);
/* Upper bound in bytes for per-chunk candidate scratch (default 8 GiB). */
int px_ctx_set_scratch_budget(px_ctx* ctx, int64_t bytes);
/* Kernels launched by this context since creation (bench.py's gpu_launches). */
int64_t px_ctx_launch_count(const px_ctx* ctx);

/* ---- per-scene / per-model state -------------------------------------------- */
/* SceneFrame planes + the observed cloud of raster.frame_to_cloud / cloud_labels
 * (raster.py:191-217), computed by the caller.  obs_src_px is (n_obs,2) (u,v).
 * If the cloud is the stride-grid cloud of this frame it is indexed as an
 * organised grid (fast path); otherwise px_search / px_cost_batch refuse it and
 * px_rendered_cost (brute force) is the path to use. */
int px_scene_upload(px_ctx* ctx, int32_t H, int32_t W, const double* depth, const uint8_t* valid,
                    const int32_t* labels, const double intr[4] /* fx fy cx cy */, int32_t stride,
                    const double* obs_points, const double* obs_lab, const int32_t* obs_src_px,
                    const int32_t* obs_labels, int64_t n_obs);
/* Same, with the observed cloud built ON THE DEVICE from the frame (replaces raster.frame_to_cloud /
 * _grid_cloud / cloud_labels, raster.py:191-217): row-major order over the valid stride-grid pixels,
 * unprojection at the pixel centre, sRGB -> Lab, label per point.  The batch path only ever reads the frame at
 * the stride-grid pixels (raster.py:263-278), so the four planes are passed already sampled there --
 * plane[::stride, ::stride], C-contiguous, GH = ceil(H/stride) rows of GW = ceil(W/stride): depth (GH,GW) float64,
 * valid (GH,GW) uint8, labels (GH,GW) int32, colour (GH,GW,3) float64 sRGB; H, W are the full image size.
 * Points, source pixels and labels are bit-identical to the host path; Lab agrees to ~1e-12.
 * n_obs_out (nullable) receives the cloud size. */
int px_scene_upload_frame(px_ctx* ctx, int32_t H, int32_t W, const double* depth_grid, const uint8_t* valid_grid,
                          const int32_t* labels_grid, const double* color_grid, const double intr[4], int32_t stride,
                          int64_t* n_obs_out);
/* Same from the FULL-resolution planes -- depth (H,W) float64, valid (H,W) uint8, labels (H,W) int32, colour (H,W,3)
 * float64, all C-contiguous: the library samples plane[::stride, ::stride] itself, into pinned staging memory (numpy's
 * strided copy of the colour plane was two thirds of the scene upload). */
int px_scene_upload_frame_full(px_ctx* ctx, int32_t H, int32_t W, const double* depth, const uint8_t* valid,
                               const int32_t* labels, const double* color, const double intr[4], int32_t stride,
                               int64_t* n_obs_out);
/* The resident observed cloud (any pointer may be NULL): points (n,3), Lab (n,3), source pixels (n,2), labels (n). */
int px_scene_download_cloud(px_ctx* ctx, double* points, double* lab, int32_t* src_px, int32_t* labels);
/* ObjectModel (model.py:75-85): mesh with colours already decoded to linear light
 * (colorspace.srgb_decode, done once per model on the host), inscribed cylinder
 * as (radius**2, z_min, z_max).  Re-uploading an id replaces it. */
int px_model_upload(px_ctx* ctx, int32_t object_id, const double* verts, const double* colors_linear,
                    const int32_t* tris, int64_t V, int64_t T, const double cyl[3]);

/* ---- raster.render_batch (raster.py:283-304) -------------------------------- */
int px_render_batch(px_ctx* ctx, const int32_t* object_ids, const double* poses3x4, int64_t n,
                    int32_t occluder_marking, double delta_occ, px_clouds** out);
int64_t px_clouds_count(const px_clouds* c);
/* counts (n) int32 */
int px_clouds_counts(px_ctx* ctx, const px_clouds* c, int32_t* counts);
/* compacted copies, sum(counts) rows each; any pointer may be NULL */
int px_clouds_download(px_ctx* ctx, const px_clouds* c, double* points, double* lab, int32_t* src_px);
/* caller-provided clouds (for m2m_gicp / cost on arbitrary LabeledClouds) */
int px_clouds_upload(px_ctx* ctx, int64_t n, const int32_t* counts, const double* points,
                     const double* lab /* nullable */, const int32_t* src_px /* nullable */, px_clouds** out);
void px_clouds_free(px_ctx* ctx, px_clouds* c);

/* raster.rasterize (raster.py:137-158) without the final sRGB encode: full-image
 * z-buffer (inf = empty), linear colour, validity and owning triangle (-1). */
int px_rasterize(px_ctx* ctx, int32_t object_id, const double pose3x4[12], double* zbuf, double* cbuf_linear,
                 uint8_t* valid, int32_t* owner);

/* ---- registration (registration.py:219-230, 514-550) ------------------------ */
/* estimate_covariances for one cloud; n must exceed k (else PX_E_ARG). */
int px_covariances(px_ctx* ctx, const double* points, int64_t n, int32_t k, double epsilon, double* cov_out);
/* Target clouds of m2m_gicp: offsets (n_targets+1), points (offsets[n],3).
 * Covariances (cfg->k_covariance, cfg->epsilon) and the nearest-neighbour grid
 * (cfg->max_correspondence_distance) are built once per distinct target on the
 * device; px_refine_batch / px_search_run must be called with the same cfg.
 * obs_index (offsets[n]) optionally gives, for every target point, its index in
 * the uploaded scene's observed cloud (ascending inside each target, as
 * search._build_targets produces, search.py:393-426): the targets are then
 * searched as organised pixel grids instead of by linear scans.  Results are
 * identical either way. */
int px_targets_upload(px_ctx* ctx, int32_t n_targets, const int64_t* offsets, const double* points,
                      const int64_t* obs_index /* nullable */, const px_gicp_cfg* cfg);
/* GICP targets cropped from the uploaded (organised) observed cloud ON THE DEVICE -- replaces
 * search._build_targets / _capsule_crop (search.py:393-426, :205-214).  3-DoF: target t is
 * { p : (px-x)^2 + (py-y)^2 + max(z_lo-pz, pz-z_hi, 0)^2 <= radius^2 } over the world-frame observed
 * points p = cam_to_world o observed, params = (n,5) rows {x, y, z_lo, z_hi, radius}; 6-DoF: target t
 * is the sub-cloud labelled object_ids[t].  Points keep ascending observed index (np.nonzero order).
 * Covariances and the search structures are built as in px_targets_upload. */
int px_targets_build_capsules(px_ctx* ctx, int32_t n_targets, const double* params, const double cam_to_world[12],
                              const px_gicp_cfg* cfg);
int px_targets_build_labels(px_ctx* ctx, int32_t n_targets, const int32_t* object_ids, const px_gicp_cfg* cfg);
/* Sizes and contents of the resident targets: offsets (n_targets+1), points (total,3) and, for
 * device-built targets, the observed index of every point (-1 for uploaded targets); any pointer may be NULL. */
int px_targets_info(px_ctx* ctx, int32_t* n_targets, int64_t* total_points);
int px_targets_download(px_ctx* ctx, int64_t* offsets, double* points, int32_t* obs_index);
int px_targets_covariances(px_ctx* ctx, double* cov_out); /* (offsets[n],9), for tests */
/* m2m_gicp: one source cloud per entry, target_idx into the uploaded targets,
 * init_T (n,12) or NULL = identity.  Outputs (any may be NULL): out_T (n,12)
 * [orthonormalised R | t], iterations, flags, rms residual, objective trace
 * (n, max_iterations, 2) with n_trace accepted steps per entry. */
int px_refine_batch(px_ctx* ctx, const px_clouds* sources, const int32_t* target_idx, const double* init_T,
                    const px_gicp_cfg* cfg, double* out_T, int32_t* out_iters, int32_t* out_flags,
                    double* out_residual, double* out_trace, int32_t* out_ntrace);

/* Test export of registration._gicp_linearize (registration.py:233-338) for ONE source / target pair at the
 * transform T, evaluated by the production kernels (source / target covariances as in registration.py:109-216, exact
 * nearest neighbours :251-261, per-point W = (Cb + R Ca R^T)^-1 and the sums in source-index order :262-338).  Outputs
 * (any may be NULL): H (36), g (6), f0, number of correspondences, corr (n) (target index or -1) and W (n,9) (zero rows
 * where no weight was formed).  Replaces the resident targets. */
int px_gicp_linearize(px_ctx* ctx, const double* src, int64_t n, const double* tgt, int64_t m, const double T[12],
                      const px_gicp_cfg* cfg, double* h36, double* g6, double* f0, int32_t* n_corr, int64_t* corr,
                      double* w);
/* Test exports of the device colour functions: colorspace.ciede2000 (colorspace.py:58-124) for n Lab pairs, and
 * colorspace.srgb_to_lab (:41-55) for n colours (linear_input != 0: linear-light input, encoded first as
 * raster.py:278 does). */
int px_ciede2000(px_ctx* ctx, const double* lab_a, const double* lab_b, int64_t n, double* out);
int px_srgb_to_lab(px_ctx* ctx, const double* rgb, int64_t n, int32_t linear_input, double* lab_out);

/* ---- cost (cost.py:91-162, search.py:189-202) -------------------------------- */
/* Per-candidate (j_o, j_r) against the uploaded organised scene.  cyl_poses
 * (n,12) = camera-frame object pose per candidate for the inscribed-cylinder
 * association, or NULL for the pixel-label association. */
int px_cost_batch(px_ctx* ctx, const px_clouds* rendered, const int32_t* object_ids, const double* cyl_poses,
                  double delta, double tau_c, int32_t use_color, int32_t* j_o, int32_t* j_r);
/* cost.rendered_cost on arbitrary clouds (brute-force exact NN, neighbors.py
 * semantics): returns j_r and the explained mask (n_obs bytes). */
int px_rendered_cost(px_ctx* ctx, const double* ren_points, const double* ren_lab, int64_t n_r,
                     const double* obs_points, const double* obs_lab, int64_t n_obs, double delta,
                     double tau_c, int32_t use_color, int32_t* j_r, uint8_t* explained);
/* neighbors.knn_full / knn_streamed: exact k nearest, ties -> lowest index;
 * idx (nq,k) int64 (-1 = missing), d2 (nq,k) (+inf = missing); k <= 32. */
int px_knn(px_ctx* ctx, const double* queries, int64_t nq, const double* targets, int64_t nt, int32_t k,
           int64_t* idx, double* d2);

/* ---- the fused search driver (search.py:268-372 for the flat candidate list) - */
/* Candidate-resident inputs.  object_ids / poses3x4 / rank_in_object are (n);
 * target_idx (n) may be NULL when cfg.refine == 0.  rank_in_object is the
 * candidate's position among its object's candidates (select_best's index). */
int px_search_upload(px_ctx* ctx, int64_t n, const int32_t* object_ids, const double* poses3x4,
                     const int32_t* target_idx, const int32_t* rank_in_object);
/* Candidates generated ON THE DEVICE from the proposal lattice (replaces the per-candidate host work of
 * search.py:240-257, proposals.py:163-210): every object's hypotheses are an outer x inner product --
 *   3-DoF: outer = grid cells (translations (n_outer,3) = x, y, fixed_z), inner = yaw spins (rotations (n_inner,9));
 *          camera pose = world_to_cam o [spin | cell] in the host BLAS rounding order (w2c_vec_order as in px_search_cfg);
 *   6-DoF: outer = rotations (n_outer,9), inner = translations (n_inner,3), already in the camera frame
 * -- with the inner index fastest and rank_in_object = outer * n_inner + inner, exactly the flat order of
 * PoseProposalSet.  Only outer items with (outer index % world) == rank are generated (the shard of one rank,
 * parallel.py:28-37's worker split; world = 1: everything).  With `gicp` non-NULL the GICP targets are built as well:
 * 3-DoF one capsule {cell x, cell y, capsule[0] = z_lo, capsule[1] = z_hi, capsule[2] = radius} per local (object, cell)
 * (search.py:407-426), 6-DoF one label sub-cloud per object.  Objects must have been uploaded (px_model_upload). */
typedef struct {
  int32_t object_id;
  int32_t n_outer, n_inner;
  const double* rotations;
  const double* translations;
  double capsule[3];
} px_lattice;
int px_search_upload_lattice(px_ctx* ctx, int32_t mode3dof, int32_t n_objects, const px_lattice* objs,
                             const double world_to_cam[12], int32_t w2c_vec_order, const double cam_to_world[12],
                             const px_gicp_cfg* gicp /* nullable: no refinement */, int32_t rank, int32_t world,
                             int64_t* n_local_out);
/* The resident candidates (any pointer may be NULL): model slot, pose (n,12), target index, rank in object. */
int px_search_candidates(px_ctx* ctx, int32_t* model_slot, double* poses3x4, int32_t* target_idx, int32_t* rank_in_object);
/* Run render -> refine -> re-render -> cost -> per-object argmin on the resident
 * candidates; results stay on the device.  Asynchronous only in the sense that
 * stage timing uses CUDA events on the context stream; returns after the last
 * kernel has been enqueued and chunk sizing has synchronised as needed. */
int px_search_run(px_ctx* ctx, const px_search_cfg* cfg);
/* Copy results to the host (any pointer may be NULL): refined candidate poses
 * (n,12), applied GICP corrections (n,12), iterations, flags, j_o, j_r, points in
 * the first / final render, packed argmin keys per uploaded model in upload
 * order ((j_o+j_r) << 32 | rank, UINT64_MAX if the model had no candidate), and
 * stage milliseconds {render, refine, rerender, cost}. */
int px_search_download(px_ctx* ctx, double* refined_poses, double* reg_T, int32_t* iters, int32_t* flags,
                       int32_t* j_o, int32_t* j_r, int32_t* n_first, int32_t* n_final,
                       uint64_t* best_key_per_model, double stage_ms[4]);
/* ---- multi-GPU: the worker fan-out of parallel.parallel_map (parallel.py:28-37) becomes one
 * process per GPU, each scoring a shard of the candidates; the ordered gather + select_best
 * (search.py:178-183, 346-372) becomes ONE NCCL all-reduce(MIN) of the packed per-object keys.
 * NCCL is bound at run time (dlopen: `nccl_path`, else the libnccl.so.2 already mapped by torch,
 * else the loader path), so libpx.so has no link-time dependency on it.
 * px_comm_unique_id: rank 0 creates the 128-byte ncclUniqueId; the host broadcasts it to the other
 * ranks (torch.distributed, MPI, a file ...); px_comm_init: every rank joins (ncclCommInitRank on
 * the context's device). */
int px_comm_unique_id(px_ctx* ctx /* nullable */, const char* nccl_path /* nullable */, uint8_t id[128]);
int px_comm_init(px_ctx* ctx, const char* nccl_path /* nullable */, const uint8_t id[128], int32_t rank, int32_t world);
int px_comm_destroy(px_ctx* ctx);
int px_comm_info(const px_ctx* ctx, int32_t* rank, int32_t* world, int32_t* nccl_version);
/* After px_search_run, enqueued on the context stream WITHOUT a host synchronisation (so that a CUDA
 * event recorded after it covers the collective): all-reduce(MIN) of the per-model packed keys across
 * the communicator (skipped when px_comm_init was not called), then the record of every model's
 * winning candidate is extracted on the device and, across ranks, delivered to every rank by an
 * all-reduce(MAX) over the records' raw 64-bit words (only the owning rank's record is non-zero).
 * The keys px_search_download returns afterwards are the global ones.  Every rank must have uploaded the same
 * models in the same order (records are indexed by model slot). */
int px_search_reduce(px_ctx* ctx);
/* Per uploaded model, in upload order (any pointer may be NULL): global packed key (UINT64_MAX = no
 * candidate), the winner's refined candidate pose (12) and applied GICP correction (12), its j_o, j_r,
 * and the largest final-render point count over all ranks' candidates of that model
 * (SearchResult.max_rendered_points, search.py:374-377).  Synchronises. */
int px_search_winners(px_ctx* ctx, uint64_t* best_key, double* refined_pose, double* reg_T, int32_t* j_o,
                      int32_t* j_r, int32_t* max_points);

/* Work counters of the last px_search_run for roofline accounting (any pointer
 * may be NULL): per candidate, the sum over GICP iterations of the
 * correspondence count, the stride-grid pixels inside the screen bounding
 * box of the first / final render, the rendered points with an observed neighbour
 * within delta and the observed points selected for the candidate (cost.py:121-152)
 * (n_c, A_g, n_m, n_fp). */
int px_search_stats(px_ctx* ctx, int32_t* ncorr_sum, int64_t* cap_first, int64_t* cap_final, int32_t* n_match,
                    int32_t* n_footprint);
/* Knife-edge log of the last px_search_run: margins[0] = min |d2 - delta^2| over every
 * rendered point's nearest observed neighbour, margins[1] = min |dE00 - tau_c| over every colour-gated match
 * (+inf when no such decision was taken).  The integer costs are exact reproductions of the reference's unless a
 * decision sits within the floating-point disagreement of the two sides (~1e-12): these two numbers show it did not. */
int px_search_knife_edges(px_ctx* ctx, double margins[2]);
/* Per-kernel timing of the GICP stage (bench.py's roofline).  When switched on, px_search_run brackets
 * every launch of the refine stage with CUDA events on the context stream; px_search_kernel_ms then
 * returns, for the last run, total milliseconds and launch counts of
 * {gicp_init, gicp_nn, gicp_step, gicp_halve, gicp_finish} (registration.py:500-511 per candidate:
 * source covariances; :251-261 nearest neighbours; :262-338 + :479-494 + :443-471 linearise, solve and
 * step halving, fused in gicp_step_kernel -- the fourth slot is only used by -DPX_GICP_SPLIT builds, which
 * run the halving as its own kernel; :473 + search.py:291-301 result and refine-apply). */
int px_ctx_set_kernel_timing(px_ctx* ctx, int32_t on);
int px_search_kernel_ms(px_ctx* ctx, double ms[5], int64_t launches[5]);
/* Number of models uploaded and their ids in slot order (for best_key_per_model). */
int px_model_count(const px_ctx* ctx);
int px_model_ids(const px_ctx* ctx, int32_t* ids);

#ifdef __cplusplus
}
#endif
#endif /* PX_H_ */
