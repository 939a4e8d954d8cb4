/*
 * voxgpr — C ABI of the B200-native voxel-GPR mapping hot path.
 *
 * Drop-in boundary for GS-LIVM's voxel mapping path as the reference package
 * `voxsplat` (/root/reference/pkg/src/voxsplat) exposes it.  The reference is
 * pure Python and has no FFI of its own; each entry point
 * below replaces one reference function or method, cited as file:line, and
 * is what a ctypes/cffi binding of that function binds.
 *
 * Conventions
 *   - plain pointers and sizes; no torch or C++ types;
 *   - every `d_` pointer is DEVICE memory, row-major, float64 unless named
 *     otherwise; `stream` is a cudaStream_t passed as void* (NULL = legacy);
 *   - every function returns VX_OK (0) or a negative VX_E_* code; the message
 *     of the last failure on the calling thread is vx_last_error();
 *   - per-voxel / per-problem outcomes are uint8 VX_ST_* codes, mapped by the
 *     host binding onto the reference exceptions (errors.py:4-46).
 *
 * All arithmetic is FP64 on the device (sm_100a); there is no CPU path.
 */
#ifndef VOXGPR_H
#define VOXGPR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VX_ABI_VERSION 1

/* return codes */
#define VX_OK 0
#define VX_E_INPUT (-1)     /* -> InputDomainError (errors.py:8)       */
#define VX_E_CONTRACT (-2)  /* -> ContractViolationError (errors.py:27)*/
#define VX_E_CUDA (-3)      /* CUDA runtime failure                     */
#define VX_E_NOMEM (-4)     /* device allocation failed                 */
#define VX_E_RANGE (-5)     /* key outside the packed 3x21-bit lattice  */
#define VX_E_CAPACITY (-6)  /* caller buffer too small; required size returned, state kept */

/* per-problem / per-voxel status */
#define VX_ST_OK 0
#define VX_ST_DEGENERATE 1  /* -> DegenerateGeometryError (errors.py:12)  */
#define VX_ST_CHOL_FAIL 2   /* -> NumericalDegeneracyError (errors.py:16) */

/* covariance kernels; SE is the reference's (gpr.py:123-130); the Matern
 * kernels are north-star extensions (parity unpinned) */
#define VX_KERNEL_SE 0
#define VX_KERNEL_MATERN32 1
#define VX_KERNEL_MATERN52 2

/* Gaussian rotation mode: identity quaternion + sqrt(diag Phi) scale is the
 * reference (splat_init.py:100-114); EIGEN (Phi = R S^2 R^T) is the
 * north-star extension (parity unpinned) */
#define VX_ROT_IDENTITY 0
#define VX_ROT_EIGEN 1

/* voxel lifecycle (voxel_map.py:118-122) */
#define VX_UNREADY 0
#define VX_READY 1
#define VX_ACTIVE 2
#define VX_CONVERGED 3

int vx_abi_version(void);
const char* vx_last_error(void);
/* number of kernel launches issued by this library so far (all threads) */
int64_t vx_launch_count(void);

/* ------------------------------------------------------------------------
 * Stateless batch entry points
 * ---------------------------------------------------------------------- */

/* voxel_keys (voxel_map.py:136-143): d_keys[i] = floor(d_xyz[i] / voxel_size)
 * as int64, true IEEE division.  VX_E_INPUT for voxel_size <= 0 or a
 * non-finite coordinate (synchronises `stream`). */
int vx_voxel_keys(const double* d_xyz, int64_t n, double voxel_size,
                  int64_t* d_keys, void* stream);

/* kernel_matrix (gpr.py:123-130): d_out[i*nb+j] = k(xa_i, xb_j); inputs (n,2). */
int vx_kernel_matrix(const double* d_xa, int64_t na, const double* d_xb, int64_t nb,
                     double lam, int32_t kernel, double* d_out, void* stream);

/* make_mesh_grid (gpr.py:104-120) for P extents (lo0,hi0,lo1,hi1):
 * d_out is (P, (n_s n_r)^2, 2), bit-exact to the reference. */
int vx_mesh_grid(const double* d_extents, int64_t num, int32_t n_s, int32_t n_r,
                 double* d_out, void* stream);

/* select_value_axis (gpr.py:57-78) for P point sets (CSR offsets, (n,3)
 * points): d_axis[p] in {0,1,2}, or -1 when degenerate (n < 3, coincident
 * or collinear -> DegenerateGeometryError). */
int vx_select_axis_batch(const double* d_points, const int64_t* d_offsets, int64_t num,
                         int8_t* d_axis, void* stream);

/* gpr_solve / gpr_solve_batch (gpr.py:173-255).  Problem p owns training
 * rows [x_off[p], x_off[p+1]) of d_x (n,2), d_f, d_noise and query rows
 * [q_off[p], q_off[p+1]) of d_xs (m,2), d_mu, d_var.  Cholesky of
 * K + diag(noise); on failure retry once with +jitter*I (gpr.py:186-194);
 * mu = Ks^T A^-1 f; var = 1 - diag(Ks^T A^-1 Ks) (unclipped).  If d_full is
 * non-NULL, Sigma* (m,m) of problem p is written at d_full[full_off[p]].
 * Status per problem in d_status.  max_n / max_m: host-known maxima. */
typedef struct {
    int64_t num_problems;
    const int64_t* d_x_off;   /* (P+1) */
    const int64_t* d_q_off;   /* (P+1) */
    const double* d_x;        /* (sum n, 2) */
    const double* d_f;        /* (sum n)    */
    const double* d_noise;    /* (sum n)    */
    const double* d_xs;       /* (sum m, 2) */
    const double* d_lam;      /* (P)        */
    double jitter;
    int32_t kernel;
    int32_t max_n;
    int32_t max_m;
    int32_t reserved;
    double* d_mu;             /* (sum m) */
    double* d_var;            /* (sum m) */
    double* d_full;           /* optional (sum m^2) */
    const int64_t* d_full_off;/* (P+1), required with d_full */
    uint8_t* d_status;        /* (P) */
} VxGprBatch;
int vx_gpr_solve_batch(const VxGprBatch* batch, void* stream);

/* init_position + init_covariance (splat_init.py:92-114) for G subgrids of
 * k points: d_pos (G,3) weighted mean, d_phi (G,3,3) weighted second moment
 * about d_center (G,3) when given, else about the weighted mean. */
int vx_subgrid_moments(const double* d_points, const double* d_weights, int64_t num,
                       int32_t k, const double* d_center, double* d_pos, double* d_phi,
                       void* stream);

/* pinhole camera (camera.py:15-76): cam = R p + t; u = fx x/z + cx ... */
typedef struct {
    double fx, fy, cx, cy;
    int32_t width, height;
    double R[9];
    double t[3];
} VxCamera;

typedef struct {
    int32_t n_s, n_r;
    double weight_floor;      /* 1e-8  (splat_init.py:24) */
    double scale_floor;       /* 1e-4  (splat_init.py:23) */
    double initial_opacity;   /* 0.5   (config.py:55)     */
    int32_t rotation_mode;    /* VX_ROT_* */
    int32_t reserved;
} VxSplatConfig;

/* caller-owned device SoA of Gaussian records (the 136-byte VXSPLAT1 record
 * split by field, formats.py:25-32): position (.,3) scale (.,3) rotation
 * (.,4) w-first, opacity (.), color SH0 (.,3), source_key (.,3) int64. */
typedef struct {
    double* position;
    double* scale;
    double* rotation;
    double* opacity;
    double* color;
    int64_t* source_key;
} VxGaussianOut;

/* init_gaussians_for_voxel (splat_init.py:134-148) over `count` predictions
 * given as SoA (count, M, 3|3|1) with M = (n_s n_r)^2, their voxel keys
 * (count,3) and an (H,W,3) float64 image; writes count*n_s^2 records at
 * out[0...].  VX_E_CONTRACT if M does not match n_s, n_r. */
int vx_gaussians_from_predictions(const double* d_pred_xyz, const double* d_pred_rgb,
                                  const double* d_pred_var, const int64_t* d_keys,
                                  int64_t count, int64_t points_per_prediction,
                                  const VxCamera* camera, const double* d_image,
                                  const VxSplatConfig* cfg, VxGaussianOut* out,
                                  void* stream);

/* ------------------------------------------------------------------------
 * Device-resident voxel map (VoxelMap, voxel_map.py:268-399)
 * ---------------------------------------------------------------------- */
typedef struct VxMap VxMap;

typedef struct {
    double voxel_size;        /* VoxelMap(voxel_size, sensor_var, tau, eta) */
    double sensor_var;
    int32_t tau;
    int32_t n_s, n_r;         /* densify grid (config.py:22-23) */
    int32_t kernel;           /* VX_KERNEL_* */
    double eta;
    double kernel_lambda;
    double jitter;
    int32_t shard_rank;       /* hash sharding: keep keys with mix(key)%world==rank */
    int32_t shard_world;      /* 1 = unsharded */
    int64_t voxel_capacity;   /* initial capacities (grown on demand) */
    int64_t point_capacity;
} VxMapConfig;

typedef struct {
    int64_t frame_index;      /* VoxelMap.frame_index after the call */
    int64_t points_in;        /* points offered */
    int64_t points_stored;    /* points kept by this shard */
    int64_t touched;          /* len(FrameUpdateSet) */
    int64_t new_voxels;
    int64_t ready_transitions;
} VxFrameInfo;

typedef struct {
    int64_t candidates;       /* READY/ACTIVE voxels of the last frame */
    int64_t solved;           /* status OK */
    int64_t degenerate;
    int64_t chol_failed;
    int64_t first_solves;     /* solved voxels that were READY (pipeline.py:145-156) */
    int64_t converged;        /* solved voxels now CONVERGED */
    int64_t max_train;        /* largest training set of the call */
} VxDensifyInfo;

/* Read-only device view of the store (valid until the next mutating call). */
typedef struct {
    int64_t num_voxels;
    const int64_t* keys;           /* (V,3) */
    const uint8_t* state;          /* (V)   VX_UNREADY.. */
    const int8_t* value_axis;      /* (V)   -1 = never solved */
    const int32_t* raw_count;      /* (V)   */
    const int64_t* raw_offset;     /* (V)   row of the voxel's first raw point */
    const int32_t* pred_slot;      /* (V)   -1 = no prediction yet */
    const uint8_t* has_pred;       /* (V)   */
    const int32_t* last_first;     /* (V)   index of the voxel's first point in the
                                              last frame that touched it (global order key
                                              for gathering sharded outputs) */
    const double* raw_xyz;         /* arena (.,3) */
    const double* raw_rgb;         /* arena (.,3) */
    int64_t pred_points;           /* M = (n_s n_r)^2 */
    const double* pred_xyz;        /* (slots, M, 3) last prediction */
    const double* pred_rgb;        /* (slots, M, 3) */
    const double* pred_var;        /* (slots, M) clipped at 0 */
    int64_t frame_touched;         /* last store_frame: voxels in first-touch order */
    const int32_t* frame_voxels;
    const uint8_t* frame_state_before;
    const uint8_t* frame_state_after;
    int64_t solve_candidates;      /* last densify: candidates in update order */
    const int32_t* solve_voxels;
    const uint8_t* solve_status;
    const uint8_t* solve_state_before;
    const uint8_t* solve_state_after;
    int64_t solved;                /* OK subset of solve_voxels, update order */
    const int32_t* solved_voxels;
    int64_t frame_index;
} VxMapView;

/* VoxelMap.__init__ / from_config (voxel_map.py:276-292) */
int vx_map_create(const VxMapConfig* cfg, VxMap** out);
int vx_map_destroy(VxMap* map);
/* drop every voxel (keeps allocations) */
int vx_map_clear(VxMap* map, void* stream);
int vx_map_view(VxMap* map, VxMapView* out);

/* VoxelMap.store_frame (voxel_map.py:313-342): hash the frame's points,
 * append them (noise := sensor_var) to their voxels in frame order, log
 * UNREADY->READY at count >= tau; the touched voxels in first-touch order
 * are frame_voxels of the view.  VX_E_INPUT on non-finite positions,
 * VX_E_RANGE outside the lattice (|key| >= 2^20). */
int vx_map_store_frame(VxMap* map, const double* d_xyz, const double* d_rgb, int64_t n,
                       VxFrameInfo* info, void* stream);

/* Input slicing for sharded maps (B200 extension): this rank
 * holds rows [global_base, global_base + n) of a scan; group them by the rank
 * that owns their voxel (mix64(key) % shard_world, the owner test of
 * vx_map_store_frame; points without a valid key go to rank 0, which reports
 * them).  d_out_xyz / d_out_rgb (n, 3) and d_out_index (n, global row numbers)
 * receive the rows grouped by owner, frame order kept within each group;
 * h_counts (HOST int64[shard_world + 1]) the group sizes, then the number of
 * rows without a valid key (already counted in rank 0's group).  After an all-to-all
 * by these counts every rank holds its voxels' points in global frame order
 * (concatenated by source rank) for vx_map_store_frame / vx_map_ingest. */
int vx_map_partition_by_owner(VxMap* map, const double* d_xyz, const double* d_rgb, int64_t n,
                              int64_t global_base, double* d_out_xyz, double* d_out_rgb,
                              int64_t* d_out_index, int64_t* h_counts, void* stream);

/* densify_frame (gpr.py:269-311) on the last frame's touched voxels: PCA
 * value axis, grid, SE Cholesky posterior, nearest colour, clip, and
 * apply_prediction (voxel_map.py:242-261,344-355).  Statuses / states in
 * the view's solve_* arrays. */
int vx_map_densify(VxMap* map, VxDensifyInfo* info, void* stream);

/* init_gaussians_for_voxel over the CURRENT predictions of `count` voxels
 * (ids from the view), camera + image as above; writes count*n_s^2 records. */
int vx_map_init_gaussians(VxMap* map, const int32_t* d_voxels, int64_t count,
                          const VxCamera* camera, const double* d_image,
                          const VxSplatConfig* cfg, VxGaussianOut* out, void* stream);

/* One ingest (pipeline.py:139-171 with expansion_threshold = 1): store,
 * densify, then Gaussians for first solves into `out` (capacity in records).
 * *out_records = records written.  camera/image may be NULL (no init).
 * camera set and out NULL: the records are deferred - the first-solve list is
 * kept, *out_records = the records it needs, and vx_map_emit_first_gaussians
 * writes them (a caller can stage the frame's image while the frame is
 * stored and solved). */
int vx_map_ingest(VxMap* map, const double* d_xyz, const double* d_rgb, int64_t n,
                  const VxCamera* camera, const double* d_image, const VxSplatConfig* cfg,
                  VxGaussianOut* out, int64_t out_capacity, int64_t* out_records,
                  VxFrameInfo* frame_info, VxDensifyInfo* densify_info, void* stream);

/* When vx_map_ingest returns VX_E_CAPACITY the frame HAS been stored and
 * densified (its voxels are ACTIVE/CONVERGED) and *out_records holds the
 * number of records its first solves need; the first-solve list is kept until
 * the next mutating call.  Grow the buffer and call this to write them
 * (pipeline.py:154-171: every first solve gets its Gaussians exactly once). */
int vx_map_emit_first_gaussians(VxMap* map, const VxCamera* camera, const double* d_image,
                                const VxSplatConfig* cfg, VxGaussianOut* out,
                                int64_t out_capacity, int64_t* out_records, void* stream);

/* `cells[key]` lookup: d_voxels[i] = voxel id of key i (-1 if absent). */
int vx_map_lookup(VxMap* map, const int64_t* d_keys, int64_t n, int32_t* d_voxels, void* stream);

/* Use an explicit update set (keys (n,3)) for the next vx_map_densify
 * instead of the last frame's (densify_frame(update_set, ...) with a set
 * that is not the latest frame).  VX_E_CONTRACT if a key is unknown. */
int vx_map_set_frame_keys(VxMap* map, const int64_t* d_keys, int64_t n, void* stream);

/* VoxelMap.apply_prediction (voxel_map.py:344-355) for a host-supplied
 * prediction of M points (device arrays); h_key is a HOST int64[3];
 * h_before_after (HOST uint8[2]) receives the state before and after.
 * VX_E_INPUT for an unknown key, VX_E_CONTRACT for a cell that is not
 * READY/ACTIVE or a size mismatch. */
int vx_map_apply_prediction(VxMap* map, const int64_t* h_key, const double* d_xyz,
                            const double* d_rgb, const double* d_var, int64_t m,
                            uint8_t* h_before_after, void* stream);

/* densify_frame's config (gpr.py:292-296): grid n_s x n_r, kernel constant,
 * jitter, kernel kind.  VX_E_CONTRACT when changing the grid size of a map
 * that already holds predictions. */
int vx_map_configure_solver(VxMap* map, int32_t n_s, int32_t n_r, double kernel_lambda,
                            double jitter, int32_t kernel);

/* init_color (splat_init.py:117-131) for n positions: SH0 of the nearest
 * pixel of each projected position, else of its fallback rgb. */
int vx_init_color(const double* d_positions, const double* d_fallback, int64_t n,
                  const VxCamera* camera, const double* d_image, double* d_sh0, void* stream);

/* read_ply (formats.py:66-147) payload decode: n binary little-endian
 * vertex records of 15 bytes (f32 x,y,z; u8 r,g,b) -> d_xyz (n,3) f64 and
 * d_rgb (n,3) f64 = u8 / 255.0.  The scan crosses PCIe at 15 B/point
 * instead of 48 B/point. */
int vx_decode_ply(const void* d_records, int64_t n, double* d_xyz, double* d_rgb, void* stream);

/* write_map (formats.py:154-169) payload: pack `count` Gaussian records from
 * SoA fields into 136-byte VXSPLAT1 records (position, scale, rotation,
 * opacity, color, source_key; little endian) at d_out (count*136 bytes). */
int vx_pack_map_records(const VxGaussianOut* records, int64_t count, void* d_out, void* stream);

/* ------------------------------------------------------------------------
 * Forward splat renderer (renderer.py): the consumer of
 * the Gaussian records.  Primitives are SoA device arrays: position (n,3),
 * scale (n,3), rotation (n,4) w-first, opacity (n), SH0 colour (n,3).
 * ---------------------------------------------------------------------- */
/* project_points (renderer.py:90-137): mean2d (n,2) pixels, cov2d (n,4)
 * row-major 2x2 with the 0.3 px^2 dilation, camera depth (n), 3-sigma radius
 * (n), valid (n) u8 (in front of near_plane, bbox on the image), bbox (n,4)
 * int64 half-open x0,x1,y0,y1 (zero when invalid). */
int vx_project_points(const double* d_pos, const double* d_scale, const double* d_rot, int64_t n,
                      const VxCamera* camera, double near_plane, double* d_mean2d, double* d_cov2d,
                      double* d_depth, double* d_radius, uint8_t* d_valid, int64_t* d_bbox,
                      void* stream);

/* render (renderer.py:184-207): front-to-back alpha blending of the valid
 * primitives (global depth order, ties by index) into colour (H,W,3), depth
 * (H,W) and silhouette (H,W), composited over black; 16x16-pixel tiles,
 * one CTA per tile. */
int vx_render(const double* d_pos, const double* d_scale, const double* d_rot, const double* d_opacity,
              const double* d_sh0, int64_t n, const VxCamera* camera, double near_plane,
              double* d_color, double* d_depth, double* d_silhouette, void* stream);

/* ------------------------------------------------------------------------
 * Measurement helper: FP64 peak of this device, max of DFMA chains and
 * m8n8k4 DMMA chains on all SMs (one shared FP64 datapath).
 * ---------------------------------------------------------------------- */
int vx_fp64_peak(double* tflops, void* stream);

/* CUDA-event timers around the library's stages, recorded on the launching
 * stream: 0 store_frame (hashing); GPR solves by training-set size bucket:
 * 1 n<=16, 2 n<=24, 6 n<=32 (warp-per-voxel DMMA kernels), 3 n<=64,
 * 7 n<=96, 4 n<=128 (DMMA tile kernels), 8 n<=160, 5 n>160 (large-n
 * kernels); 9 Gaussian init, 10 whole densify, 11 PCA prepass.  vx_profile(1) resets
 * and enables; vx_profile_read fills total ms and launch counts per stage
 * and returns the number of stages. */
int vx_profile(int enable);
int vx_profile_read(double* ms, int64_t* launches, int32_t max_stages);

#ifdef __cplusplus
}
#endif
#endif /* VOXGPR_H */
