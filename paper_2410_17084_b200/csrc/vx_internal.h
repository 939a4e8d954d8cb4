// Host-side internals shared by the voxgpr translation units.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "../../include/voxgpr.h"

namespace vx {

void set_error(const char* fmt, ...);
extern std::atomic<int64_t> g_launches;
inline void count_launch(int k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

#define VX_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            ::vx::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #call,            \
                            cudaGetErrorString(e_));                               \
            return e_ == cudaErrorMemoryAllocation ? VX_E_NOMEM : VX_E_CUDA;       \
        }                                                                          \
    } while (0)

#define VX_CHECK_LAUNCH() VX_CUDA(cudaGetLastError())

#define VX_TRY(expr)              \
    do {                          \
        int r_ = (expr);          \
        if (r_ != VX_OK) return r_; \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Optional CUDA-event timers around the library's stages (vx_profile_*).
enum ProfStage { P_HASH = 0, P_GPR_B0, P_GPR_B1, P_GPR_B2, P_GPR_B3, P_GPR_B4, P_GPR_B5, P_GPR_B6, P_GPR_B7, P_SPLAT, P_DENSIFY, P_PCA, P_COUNT };
void prof_begin(int stage, cudaStream_t s);
void prof_end(int stage, cudaStream_t s);

int sm_count();

// ---------------------------------------------------------------- scratch
// Grow-only device buffer.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    int reserve(size_t want, cudaStream_t s, bool keep = false);
    template <typename T> T* as() const { return static_cast<T*>(ptr); }
    void release();
};

// ---------------------------------------------------------------- scan/sort
// exclusive prefix sums; `total` (device, may be null) receives the sum.
int scan_exclusive_i32(const int32_t* in, int32_t* out, int64_t n, int32_t* total,
                       DevBuf& tmp, cudaStream_t s);
int scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total,
                       DevBuf& tmp, cudaStream_t s);
// stable LSD radix sort of (key, value) pairs by the low `bits` bits of key;
// vals_identity: the values are 0..n-1, generated instead of read
int map_partition_by_owner(VxMap* m, const double* xyz, const double* rgb, int64_t n,
                           int64_t gbase, double* oxyz, double* orgb, int64_t* ogidx,
                           int64_t* h_counts, cudaStream_t s);
int radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                     int64_t n, int bits, DevBuf& tmp, cudaStream_t s, bool* result_in_alt,
                     bool vals_identity = false);

// ---------------------------------------------------------------- GPR
// Voxel-mode work description shared by the GPR kernels (device pointers).
struct VoxelSolveArgs {
    // work list
    const int32_t* items;      // indices s into the candidate arrays
    int32_t num_items;
    const int32_t* cand_voxel; // (S) voxel id per candidate
    const int32_t* cand_n;     // (S) training size
    uint8_t* cand_status;      // (S)
    uint8_t* cand_before;      // (S)
    uint8_t* cand_after;       // (S)
    int8_t* cand_axis;         // (S) value axis from the PCA prepass, -1 degenerate
    double* cand_meanf;        // (S) pairwise mean of the targets
    // store
    const int64_t* keys;       // (V,3)
    uint8_t* state;
    int8_t* value_axis;
    const int32_t* raw_count;
    const int64_t* raw_offset;
    const int32_t* pred_slot;
    uint8_t* has_pred;
    const double* raw_xyz;
    const double* raw_rgb;
    double* pred_xyz;
    double* pred_rgb;
    double* pred_var;
    // config
    double voxel_size, sensor_var, eta, lam, jitter;
    int n_s, n_r, kernel;
    int M;                     // (n_s n_r)^2
};

int launch_voxel_solve(const VoxelSolveArgs& a, int max_n, DevBuf& work, cudaStream_t s,
                       int bucket);
int launch_problem_solve(const VxGprBatch& b, const int32_t* d_items, int32_t count,
                         int max_n, int max_m, DevBuf& work, cudaStream_t s, int bucket);

// bucket boundaries for the training-set size n: warp kernels for n <= 16,
// 32, 64; the blocked CTA kernel for n <= 128 (shared-memory resident) and
// beyond (shared memory when it fits, else an L2-resident workspace)
// ids: 0 n<=16, 1 n<=24, 5 n<=32 (warp kernels), 2 n<=64, 6 n<=96, 3 n<=128,
// 7 n<=160 (DMMA tile kernels), 4 n>160 (CTA kernel); later buckets got
// higher ids so the profiling stage ids of earlier ones stay stable
constexpr int NUM_BUCKETS = 8;
__host__ __device__ inline int bucket_of(int n) {
    return n <= 16 ? 0
         : n <= 24 ? 1
         : n <= 32 ? 5
         : n <= 64 ? 2
         : n <= 96 ? 6
         : n <= 128 ? 3
         : n <= 160 ? 7 : 4;
}
int launch_pca_prepass(const VoxelSolveArgs& a, int S, long long* bucket_counts, cudaStream_t s);
int launch_bucket_items(const VoxelSolveArgs& a, int S, int32_t* items, const long long* base,
                        long long* fill, cudaStream_t s);

// ---------------------------------------------------------------- splat init
int launch_gaussians(const double* pred_xyz, const double* pred_rgb, const double* pred_var,
                     const int32_t* slot_of, const int32_t* voxel_ids, const int64_t* keys,
                     const int64_t* direct_keys, int64_t count, int M, const VxCamera& cam,
                     const double* image, const VxSplatConfig& cfg, const VxGaussianOut& out,
                     cudaStream_t s);
int launch_decode_ply(const uint8_t* rec, int64_t n, double* xyz, double* rgb, cudaStream_t s);

// ---------------------------------------------------------------- renderer
int project_points(const double* pos, const double* scale, const double* rot, int64_t n,
                   const VxCamera& cam, double near, double* mean2d, double* cov2d, double* depth,
                   double* radius, uint8_t* valid, int64_t* bbox, cudaStream_t s);
int render_splats(const double* pos, const double* scale, const double* rot, const double* opacity,
                  const double* sh0, int64_t n, const VxCamera& cam, double near, double* color,
                  double* depth, double* sil, cudaStream_t s);
int launch_pack_records(const VxGaussianOut& in, int64_t count, void* out, cudaStream_t s);
int launch_moments(const double* pts, const double* w, int64_t G, int k, const double* center,
                   double* pos, double* phi, cudaStream_t s);

}  // namespace vx
