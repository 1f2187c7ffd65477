/*
 * refusion_b200.h — C ABI of the B200-native ReFusion hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++/torch types.
 * Each entry point replaces one interface of the CPU reference (`tsdfslam`,
 * /root/reference/proj/include/tsdfslam); the reference symbol it replaces is
 * cited beside it. Conventions shared by every call:
 *
 *  - Poses are 12 doubles, camera-to-world: rotation row-major (9) then
 *    translation (3) — `Pose` (geometry.hpp:69-108).
 *  - Images are dense row-major W*H: depth f32 metres (<= 0 or non-finite =
 *    invalid, image.hpp:66-68), colour RGB8 (3 bytes/pixel), masks u8
 *    (nonzero = excluded, image.hpp:71).
 *  - A NULL mask means "no mask" (the reference's `const PixelMask* = nullptr`).
 *  - Voxels are 8 bytes {f32 sdf, u8 weight, u8 r, u8 g, u8 b}
 *    (tsdf_volume.hpp:32-37); a brick is 8^3 voxels, x fastest.
 *  - Every call returns an rf_status; on failure rf_last_error() holds a
 *    thread-local message. The C++ host layer rethrows RF_TRACKING_LOST as
 *    TrackingLostError, RF_RESOURCE_LIMIT as ResourceLimitError and
 *    RF_INVALID_ARGUMENT as std::invalid_argument (errors.hpp:9-21).
 *  - Calls are synchronous like the reference (results are on the host when
 *    they return). Handles are not thread-safe, matching the reference's
 *    volume concurrency contract (tsdf_volume.hpp:64-66).
 *  - Device-memory inputs (rf_frame.memory == RF_MEMORY_DEVICE, and the
 *    device-pointer variants of the evaluation calls) are read on the
 *    library's own CUDA streams, which are not ordered after the caller's
 *    streams: the work that produced them must be complete when the call is
 *    made (synchronise the producing stream first; the Python layer does).
 *    rf_pipeline_stream() exposes the pipeline's stream for callers that want
 *    to order against it with events instead.
 *  - block_side must be 8 (the reference default); other values return
 *    RF_UNSUPPORTED.
 */
#ifndef REFUSION_B200_H
#define REFUSION_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RF_OK = 0,
    RF_INVALID_ARGUMENT = 1,
    RF_TRACKING_LOST = 2,   /* TrackingLostError (errors.hpp:14) */
    RF_RESOURCE_LIMIT = 3,  /* ResourceLimitError (errors.hpp:19) */
    RF_CUDA_ERROR = 4,
    RF_IO_ERROR = 5,
    RF_UNSUPPORTED = 6,
    RF_FAILED = 7           /* any other std::runtime_error of the reference */
} rf_status;

enum { RF_MEMORY_HOST = 0, RF_MEMORY_DEVICE = 1 };

/* CameraIntrinsics (geometry.hpp:11-38) */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double depth_scale;
} rf_intrinsics;

/* VolumeConfig (tsdf_volume.hpp:14-29); hash_capacity 0 = next power of two
 * >= 4/3 * max_blocks (the load bound of spatial_hash.hpp:51), at least 2^18
 * (an overflowing allocation holds its not-yet-numbered keys in the table). */
typedef struct {
    double voxel_size, truncation;
    int32_t block_side, max_weight, carve_weight, reserved0;
    double min_depth, max_depth, carve_clip;
    uint64_t max_blocks;
    uint64_t hash_capacity;
} rf_volume_config;

/* RegistrationConfig (registration.hpp:13-23); `threads` is accepted and ignored.
 * Extension (not in the reference, off by default): Huber weighting of the
 * depth (huber_depth, metres) and colour (huber_color, scaled intensity)
 * residuals in the LM normal equations and cost; 0 = plain least squares as
 * the reference (registration.cpp:72-95), bit for bit. */
typedef struct {
    double color_weight;
    int32_t pyramid_levels, max_iterations;
    double lm_lambda_init, lm_lambda_up, lm_lambda_down, convergence_eps;
    int32_t min_valid_residuals, threads;
    double huber_depth, huber_color;
} rf_registration_config;

/* MaskConfig (dynamics_mask.hpp:10-17).
 * Extension (not in the reference, off by default): free_space > 0 also
 * seeds the mask with pixels whose measured point lies at least free_space
 * metres in front of the model surface (signed residual > free_space: the
 * model holds that space as free). 0 = the reference's threshold, bit for bit.
 * The residual images then carry the sign in bit 1 of `valid` (3 = valid and
 * positive); rf_mask_stages reads it the same way. */
typedef struct {
    double gamma, truncation, theta;
    int32_t erode_radius, dilate_radius, connectivity, reserved0;
    double free_space;
} rf_mask_config;

/* PipelineConfig (config.hpp:12-24) with RefinementConfig (depth_refinement.hpp:12-17) */
typedef struct {
    rf_volume_config volume;
    rf_registration_config registration;
    rf_mask_config mask;
    int32_t refine_enabled, refine_window;
    double far_value;
    int32_t bisection_iterations, dynamics_enabled, threads, reserved0;
} rf_pipeline_config;

/* One RGB-D measurement, `Frame` (image.hpp:94-103). memory = RF_MEMORY_HOST
 * (pointers are copied in, pinned memory is fastest) or RF_MEMORY_DEVICE
 * (device pointers of the volume's GPU, read in place). rgb may be NULL. */
typedef struct {
    const float* depth;
    const uint8_t* rgb;
    rf_intrinsics intrinsics;
    double timestamp;
    int32_t memory;
    int32_t reserved0;
} rf_frame;

/* FrameStats (pipeline.hpp:18-29) */
typedef struct {
    uint64_t frame_index;
    double timestamp;
    int32_t tracking_lost, converged, registrations, iterations;
    uint64_t valid_residuals, masked_pixels;
    double final_error, runtime_ms;
} rf_frame_stats;

/* RegistrationResult (registration.hpp:66-74); residual images are separate out-params */
typedef struct {
    double pose[12];
    int32_t converged, iterations;
    uint64_t valid_residuals;
    double final_error;
} rf_registration_result;

/* LinearizeResult (registration.hpp:47-55) */
typedef struct {
    double H[36];
    double b[6];
    double depth_error, color_error, error;
    uint64_t valid_count;
    int32_t degenerate, reserved0;
} rf_linearize_result;

/* Per-frame work counters for the algorithmic-bytes model (not in the reference). */
typedef struct {
    uint64_t dda_visits, new_blocks, visible_bricks, num_blocks;
    int32_t floodfill_rounds, overflow;
    int32_t passes, reserved0;  /* Accumulate passes of the frame's registrations */
    double pixel_passes;        /* sum of the pixel counts of those passes */
} rf_frame_counters;

typedef struct rf_volume rf_volume;
typedef struct rf_pipeline rf_pipeline;
typedef struct rf_mesh rf_mesh;

const char* rf_last_error(void);
const char* rf_version(void);

/* ---- volume: TsdfVolume (tsdf_volume.hpp:67-134) ---------------------- */
rf_status rf_volume_create(const rf_volume_config* cfg, int device, rf_volume** out);      /* TsdfVolume(VolumeConfig) */
void rf_volume_destroy(rf_volume* v);
rf_status rf_volume_num_blocks(const rf_volume* v, uint64_t* out);                         /* num_blocks() */
rf_status rf_volume_hash_capacity(const rf_volume* v, uint64_t* out);
rf_status rf_volume_get_config(const rf_volume* v, rf_volume_config* out);                 /* config() */
rf_status rf_volume_allocate_blocks(rf_volume* v, const int32_t* coords, uint64_t n,
                                    int32_t* created);                                     /* AllocateBlock (batched) */
rf_status rf_volume_allocate_for_frame(rf_volume* v, const rf_frame* f, const double pose[12],
                                       const uint8_t* mask);                               /* AllocateForFrame */
rf_status rf_volume_integrate(rf_volume* v, const rf_frame* f, const double pose[12],
                              const uint8_t* mask);                                        /* Integrate */
rf_status rf_volume_carve(rf_volume* v, const rf_frame* f, const double pose[12]);         /* CarveFreeSpace */
/* mode 0 SampleSdf, 1 SampleIntensity, 2 SampleSdfWithGradient,
 * 3 SampleIntensityWithGradient, 4 SampleSdfGradient. grad may be NULL. */
rf_status rf_volume_sample(const rf_volume* v, int32_t mode, const double* points, uint64_t n,
                           double* value, double* grad, uint8_t* valid);
rf_status rf_volume_get_voxels(const rf_volume* v, const int32_t* voxel_coords, uint64_t n,
                               uint8_t* voxels, uint8_t* found);                          /* const VoxelHandle */
rf_status rf_volume_set_voxels(rf_volume* v, const int32_t* voxel_coords, uint64_t n,
                               const uint8_t* voxels, uint64_t* missing);                 /* mutable VoxelHandle */
/* blocks() in pool (allocation) order; voxels may be NULL. capacity in blocks. */
rf_status rf_volume_export_blocks(const rf_volume* v, int32_t* coords, uint8_t* voxels, uint64_t capacity,
                                  uint64_t* count);
rf_status rf_volume_hash_occupancy(const rf_volume* v, uint8_t* bitmap);                  /* hash_capacity bytes */
/* FindBlock (tsdf_volume.cpp:59-62): one hash probe on the device and one brick
 * copied back; *found = 0 when the block is not allocated. voxels (512 x 8 B,
 * x fastest) may be NULL. */
rf_status rf_volume_find_block(const rf_volume* v, const int32_t block_coord[3], uint8_t* voxels, int32_t* found);
/* Writes one allocated brick's 512 voxels (the write-back of the host layer's
 * mutable VoxelHandle mirror, tsdf_volume.cpp:89-91); *found = 0 when absent. */
rf_status rf_volume_write_block(rf_volume* v, const int32_t block_coord[3], const uint8_t* voxels, int32_t* found);
rf_status rf_volume_reset(rf_volume* v);
rf_status rf_volume_save(const rf_volume* v, const char* path);                           /* Save (TSDFVOL v1) */
rf_status rf_volume_load(const char* path, int device, rf_volume** out);                  /* Load */

/* ---- registration (registration.hpp:42-85) ----------------------------- */
/* BuildPyramid (registration.hpp:42, registration.cpp:119-182) on the GPU.
 * Outputs hold all levels back to back, level 0 first; level l has
 * (width >> l) * (height >> l) pixels. depth: f32; intensity: f32, ToIntensity
 * at level 0 then 2x2 means (requires f->rgb); mask_out: u8, any-of-2x2
 * (requires mask). Any output may be NULL; k_out (levels records) receives
 * CameraIntrinsics::Scaled(l). RF_INVALID_ARGUMENT when a level is empty. */
rf_status rf_build_pyramid(const rf_frame* f, const uint8_t* mask, int32_t levels, int device, float* depth,
                           float* intensity, uint8_t* mask_out, rf_intrinsics* k_out);
rf_status rf_linearize(const rf_volume* v, const rf_frame* f, const double pose[12],
                       const rf_registration_config* cfg, const uint8_t* mask, rf_linearize_result* out);
rf_status rf_evaluate_depth_error(const rf_volume* v, const rf_frame* f, const double pose[12],
                                  const uint8_t* mask, double* error, float* res_sq, uint8_t* res_valid);
rf_status rf_evaluate_color_error(const rf_volume* v, const rf_frame* f, const double pose[12],
                                  const uint8_t* mask, double* error);
rf_status rf_register(const rf_volume* v, const rf_frame* f, const double initial_pose[12], const uint8_t* mask,
                      const rf_registration_config* cfg, rf_registration_result* out, float* res_sq,
                      uint8_t* res_valid);                                                 /* Register */

/* ---- dynamics mask (dynamics_mask.hpp:21-41) ----------------------------
 * stages: bit0 ThresholdResiduals, bit1 Erode, bit2 FloodfillDepth, bit3 Dilate
 * (15 = BuildMask). With bit0 clear, `res_valid` is read as the input mask;
 * `res_sq` may be NULL without bit0, `depth` without bit2. */
rf_status rf_mask_stages(const float* res_sq, const uint8_t* res_valid, const float* depth, int32_t width,
                         int32_t height, const rf_mask_config* cfg, int32_t stages, int device, uint8_t* out,
                         uint64_t* masked);

/* ---- raycast (ray-march of RenderVirtualDepth, depth_refinement.cpp:32-79) */
rf_status rf_raycast(const rf_volume* v, const double view_pose[12], const rf_intrinsics* k,
                     int32_t bisection_iterations, float* out_depth);

/* ---- depth refinement (depth_refinement.hpp:46-57) ----------------------
 * RenderVirtualDepth over a window of n frames (their poses, masks[i] may be
 * NULL, masks itself may be NULL) seen from view_pose with intrinsics k, in a
 * fresh volume of config vcfg; RefineDepth of frames[0] into refined_depth
 * when it is non-NULL. */
rf_status rf_render_virtual_depth(const rf_frame* frames, const double* poses, const uint8_t* const* masks, int32_t n,
                                  const double view_pose[12], const rf_intrinsics* k, const rf_volume_config* vcfg,
                                  int32_t bisection_iterations, double far_value, int device, float* virtual_depth,
                                  float* refined_depth);

/* ---- mesh: ExtractMesh / WritePly (mesh.hpp:14-29) -----------------------
 * The mesh stays on the device; vertices f32 xyz, colours RGB8, faces i32
 * triples, in the reference's exact order (blocks sorted by x, y, z). */
rf_status rf_volume_extract_mesh(const rf_volume* v, int32_t min_weight, rf_mesh** out);   /* ExtractMesh */
rf_status rf_mesh_counts(const rf_mesh* m, uint64_t* vertices, uint64_t* faces);
rf_status rf_mesh_copy(const rf_mesh* m, float* xyz, uint8_t* rgb, int32_t* faces);       /* host; any may be NULL */
rf_status rf_mesh_device_buffers(const rf_mesh* m, const float** xyz, const uint8_t** rgb, const int32_t** faces);
rf_status rf_mesh_write_ply(const rf_mesh* m, const char* path);                          /* WritePly */
void rf_mesh_destroy(rf_mesh* m);

/* ---- evaluation (evaluation.hpp:12-50) ----------------------------------
 * Trajectories are n timestamps plus 12 n pose doubles (camera-to-world).
 * Point clouds are f32 xyz triples; `memory` says whether queries, reference
 * and out (NearestDistances) or distances (DistanceCdf) are host or device
 * pointers. Bin edges and the CDF are host arrays. */
rf_status rf_ate_rmse(const double* est_t, const double* est_poses, uint64_t n_est, const double* gt_t,
                      const double* gt_poses, uint64_t n_gt, double max_dt, double* rmse, double alignment[12],
                      uint64_t* pairs);                                                    /* AteRmse; < 3 pairs: RF_FAILED */
rf_status rf_rpe_over_time(const double* est_t, const double* est_poses, uint64_t n_est, const double* gt_t,
                           const double* gt_poses, uint64_t n_gt, double delta, double max_dt, double* timestamps,
                           double* errors, uint64_t capacity, uint64_t* count);            /* RpeOverTime */
rf_status rf_nearest_distances(const float* queries, uint64_t nq, const float* reference, uint64_t nr, int32_t memory,
                               int device, double* out);                                  /* NearestDistances */
rf_status rf_distance_cdf(const double* distances, uint64_t n, int32_t memory, int device, const double* edges,
                          uint64_t ne, double* cdf);                                       /* DistanceCdf */

/* ---- pipeline (pipeline.hpp:51-96) ------------------------------------- */
rf_status rf_pipeline_create(const rf_pipeline_config* cfg, int device, rf_pipeline** out);
void rf_pipeline_destroy(rf_pipeline* p);
rf_status rf_pipeline_process_frame(rf_pipeline* p, const rf_frame* f, rf_frame_stats* stats,
                                    double pose_out[12]);                                  /* ProcessFrame */
/* ProcessFrame over n frames with the GPU work of up to 64 frames enqueued back to back
 * (RunSequence, pipeline.cpp:137-145, without a host round trip per frame). stats
 * (n records) and poses (12 n doubles) may be NULL. Host frames must stay valid for the
 * call. With refinement, profiling or tracing on, the frames are processed one by one. */
rf_status rf_pipeline_process_frames(rf_pipeline* p, const rf_frame* frames, uint64_t n, rf_frame_stats* stats,
                                     double* poses);
rf_status rf_pipeline_finalize(rf_pipeline* p);                                            /* Finalize */
rf_status rf_pipeline_volume(rf_pipeline* p, rf_volume** out);                             /* volume() (borrowed) */
rf_status rf_pipeline_tracking_losses(const rf_pipeline* p, uint64_t* out);               /* tracking_losses() */
rf_status rf_pipeline_trajectory(const rf_pipeline* p, double* timestamps, double* poses, uint64_t capacity,
                                 uint64_t* count);                                         /* trajectory() */
rf_status rf_pipeline_last_mask(const rf_pipeline* p, uint8_t* out, int32_t* has_mask);    /* FrameDebug::mask */
rf_status rf_pipeline_last_residuals(const rf_pipeline* p, float* res_sq, uint8_t* res_valid); /* FrameDebug::residuals */
rf_status rf_pipeline_last_counters(const rf_pipeline* p, rf_frame_counters* out);
/* Refinement window (refine_enabled): frames waiting for integration, and the
 * FrameDebug::virtual_depth / refined_depth of the last IntegrateFront. The
 * pipeline ray-marches only raw-depth holes unless debug images are enabled;
 * virtual_depth requires them. */
rf_status rf_pipeline_window_size(const rf_pipeline* p, uint64_t* out);
rf_status rf_pipeline_finalize_one(rf_pipeline* p);  /* one IntegrateFront of Finalize (no-op when empty) */
rf_status rf_pipeline_set_debug_images(rf_pipeline* p, int32_t enable);
rf_status rf_pipeline_last_refinement(const rf_pipeline* p, float* virtual_depth, float* refined_depth,
                                      uint64_t* frame_index, int32_t* has);
/* Per-stage device time with CUDA events on the pipeline's stream (off by
 * default). stage_ms[0..3] = track (k_track: pyramid + LM + mask), allocate,
 * cull, fuse (carve+integrate), accumulated over `frames` frames since the
 * last enable; `launches` counts every kernel this pipeline launched. */
rf_status rf_pipeline_set_profiling(rf_pipeline* p, int32_t enable);
rf_status rf_pipeline_stage_times(const rf_pipeline* p, double stage_ms[4], uint64_t* frames, uint64_t* launches);
/* Sums of the per-frame counters over the frames profiled since the last enable. */
rf_status rf_pipeline_profile_counters(const rf_pipeline* p, rf_frame_counters* sums);
rf_status rf_pipeline_stream(const rf_pipeline* p, void** cuda_stream);                   /* cudaStream_t */

/* ---- synthetic input (synth.cpp:136-203 on the GPU; workload generator) ----
 * prims: array of rf_synth_primitive records (176 bytes each, see
 * paper_1905_02082_b200/synth.py) with world-to-object poses for this frame;
 * outputs are device buffers on `device`. */
/* ---- diagnostics ----------------------------------------------------------
 * Cost of one grid-wide barrier (reduce = 0) or barrier + 30-value
 * deterministic all-reduce (reduce = 1) of the persistent tracking kernel. */
rf_status rf_diag_grid_barrier(int device, int32_t iters, int32_t reduce, double* us_per_call);
/* SM cycles of one LM step on one thread: [solve, ExpMap + compose, total]. */
rf_status rf_diag_pass_bench(rf_volume* v, const rf_frame* f, const double pose[12], int32_t level, int32_t iters,
                             double color_weight, double* us_per_pass, double* acc);  /* acc: 30 doubles or NULL */
rf_status rf_diag_lm_step(int device, int32_t iters, double cycles[3]);
/* Structural invariants of a volume, as error counts (all zero when consistent):
 * [0] occupied slots with a value that is neither a brick nor pending, [1] bricks
 * whose slot does not hold their key and index, [2] duplicated keys, [3] link
 * records that disagree with a hash probe, [4] pending (claimed, unnumbered) keys. */
rf_status rf_diag_volume_check(const rf_volume* v, uint64_t errors[5]);

rf_status rf_synth_render(const void* prims, int32_t nprims, const double cam_pose[12], const rf_intrinsics* k,
                          double noise_sigma_scale, double dropout, uint64_t seed, uint64_t frame_index,
                          float* depth, uint8_t* rgb, uint8_t* labels, int device);

/* ---- memory helpers ------------------------------------------------------ */
void* rf_host_alloc(size_t bytes);  /* pinned host memory (fast frame uploads) */
void rf_host_free(void* p);
void* rf_device_alloc(size_t bytes, int device);
void rf_device_free(void* p);
rf_status rf_copy_to_device(void* dst, const void* src, size_t bytes);

#ifdef __cplusplus
}
#endif

#endif /* REFUSION_B200_H */
