// extern "C" entry points of libvoxgpr (include/voxgpr.h) and the small
// stateless kernels behind them.
#include <cstdarg>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "vx_common.cuh"
#include "vx_internal.h"

namespace vx {

std::atomic<int64_t> g_launches{0};
static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int sm_count() {
    static int cached = 0;
    if (cached == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
    }
    return cached;
}

int DevBuf::reserve(size_t want, cudaStream_t s, bool keep) {
    if (want <= bytes) return VX_OK;
    size_t nb = want + want / 4 + 256;
    void* p = nullptr;
    VX_CUDA(cudaMalloc(&p, nb));
    if (keep && ptr && bytes) VX_CUDA(cudaMemcpyAsync(p, ptr, bytes, cudaMemcpyDeviceToDevice, s));
    if (ptr) VX_CUDA(cudaFree(ptr));
    ptr = p;
    bytes = nb;
    return VX_OK;
}

void DevBuf::release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
}

// ------------------------------------------------------------ small kernels
__global__ void k_voxel_keys(const double* xyz, int64_t n, double vs, int64_t* keys, int* err) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * 3) return;
    const double v = xyz[i];
    if (!isfinite(v)) {
        atomicOr(err, 1);
        keys[i] = 0;
        return;
    }
    const double f = floor(xdiv(v, vs));
    if (!(f >= -9.2233720368547758e18 && f < 9.2233720368547758e18)) {
        atomicOr(err, 2);
        keys[i] = 0;
        return;
    }
    keys[i] = int64_t(f);
}

__global__ void k_kernel_matrix(const double* xa, int64_t na, const double* xb, int64_t nb, double lam,
                                int kind, double* out) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= na * nb) return;
    const int64_t i = e / nb, j = e - i * nb;
    out[e] = kernel_value(kind, lam, dist2_exact(xa[i * 2], xa[i * 2 + 1], xb[j * 2], xb[j * 2 + 1]));
}

// make_mesh_grid (gpr.py:104-120): c_i = lo + ((i + 0.5) * (hi - lo)) / m,
// ordered (subgrid row, subgrid col, fine row, fine col)
__global__ void k_mesh_grid(const double* ext, int64_t P, int n_s, int n_r, double* out) {
    const int mm = n_s * n_r;
    const int64_t M = int64_t(mm) * mm;
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= P * M) return;
    const int64_t p = e / M;
    const int q = int(e - p * M);
    const int nr2 = n_r * n_r;
    const int sr = q / (n_s * nr2);
    const int rem = q - sr * n_s * nr2;
    const int sc = rem / nr2;
    const int rem2 = rem - sc * nr2;
    const int fr = rem2 / n_r, fc = rem2 - fr * n_r;
    const double lo0 = ext[p * 4], hi0 = ext[p * 4 + 1], lo1 = ext[p * 4 + 2], hi1 = ext[p * 4 + 3];
    out[e * 2] = xadd(lo0, xdiv(xmul(double(sr * n_r + fr) + 0.5, xsub(hi0, lo0)), double(mm)));
    out[e * 2 + 1] = xadd(lo1, xdiv(xmul(double(sc * n_r + fc) + 0.5, xsub(hi1, lo1)), double(mm)));
}

// select_value_axis (gpr.py:57-78), one thread per point set (pca_value_axis)
__global__ void k_select_axis(const double* pts, const int64_t* off, int64_t P, int8_t* axis_out) {
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int64_t b = off[p];
    const double* P3 = pts + b * 3;
    axis_out[p] = int8_t(pca_value_axis([&](int r) { return P3 + int64_t(r) * 3; },
                                        int(off[p + 1] - b)));
}

// problem-mode bucketing for gpr_solve_batch
__global__ void k_problem_buckets(const int64_t* x_off, int64_t P, int32_t* items, int* fill,
                                  const int* base) {
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int n = int(x_off[p + 1] - x_off[p]);
    const int b = bucket_of(n);
    const int pos = atomicAdd(fill + b, 1);
    items[base[b] + pos] = int32_t(p);
}
__global__ void k_problem_count(const int64_t* x_off, int64_t P, int* counts) {
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= P) return;
    atomicAdd(counts + bucket_of(int(x_off[p + 1] - x_off[p])), 1);
}

// FP64 peak: independent DFMA chains, 8 per thread
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = fma(r[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += r[k];
    if (s == 12345.678) out[0] = s;
}

// FP64 tensor-core (m8n8k4 DMMA) throughput: 8 independent accumulator chains
// per warp; the solve kernels' inner products run on this pipe
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, int iters, double a, double b) {
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3 + k;
    const double x = a + threadIdx.x * 1e-12, y = b;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(x), "d"(y));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[0] = s;
}

// ---------------------------------------------------------------- profiling
struct ProfState {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[P_COUNT];
    cudaEvent_t open[P_COUNT] = {};
    double ms[P_COUNT] = {};
    int64_t n[P_COUNT] = {};
};
static ProfState g_prof;
static std::mutex g_prof_mu;

void prof_begin(int stage, cudaStream_t s) {
    if (!g_prof.on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    g_prof.open[stage] = e;
}

void prof_end(int stage, cudaStream_t s) {
    if (!g_prof.on || !g_prof.open[stage]) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.ev[stage].push_back({g_prof.open[stage], e});
    g_prof.open[stage] = nullptr;
}

static void prof_collect() {
    for (int k = 0; k < P_COUNT; ++k) {
        for (auto& pr : g_prof.ev[k]) {
            float ms = 0;
            cudaEventSynchronize(pr.second);
            cudaEventElapsedTime(&ms, pr.first, pr.second);
            g_prof.ms[k] += ms;
            g_prof.n[k] += 1;
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
        g_prof.ev[k].clear();
    }
}

struct Scratch {
    DevBuf a, b, c;
    int* host = nullptr;
};
static std::mutex g_scratch_mu;
static Scratch& scratch() {
    static Scratch s;
    return s;
}

}  // namespace vx

using namespace vx;

// map internals (vx_map.cu)
namespace vx {
int map_store_frame(VxMap* m, const double* xyz, const double* rgb, int64_t n, VxFrameInfo* info,
                    cudaStream_t s);
int map_densify(VxMap* m, VxDensifyInfo* info, cudaStream_t s);
int map_ingest(VxMap* m, const double* xyz, const double* rgb, int64_t n, const VxCamera* cam,
               const double* image, const VxSplatConfig* scfg, VxGaussianOut* out,
               int64_t out_capacity, int64_t* out_records, VxFrameInfo* fi, VxDensifyInfo* di,
               cudaStream_t s);
int map_emit_first_gaussians(VxMap* m, const VxCamera* cam, const double* image,
                             const VxSplatConfig* scfg, VxGaussianOut* out, int64_t out_capacity,
                             int64_t* out_records, cudaStream_t s);
int map_clear(VxMap* m, cudaStream_t s);
int map_lookup(VxMap* m, const int64_t* keys, int64_t n, int32_t* out, cudaStream_t s);
int map_set_frame_keys(VxMap* m, const int64_t* keys, int64_t n, cudaStream_t s);
int map_apply_prediction(VxMap* m, const int64_t* h_key, const double* xyz, const double* rgb,
                         const double* var, int64_t M, uint8_t* h_before_after, cudaStream_t s);
int map_configure_solver(VxMap* m, int n_s, int n_r, double lam, double jitter, int kernel);
int launch_init_color(const double* pos, const double* fallback, int64_t n, const VxCamera& cam,
                      const double* image, double* out, cudaStream_t s);
VxMap* map_new(const VxMapConfig& cfg, int* rc);
void map_delete(VxMap* m);
void map_fill_view(VxMap* m, VxMapView* v);
int map_init_gaussians(VxMap* m, const int32_t* vids, int64_t count, const VxCamera& cam,
                       const double* image, const VxSplatConfig& cfg, const VxGaussianOut& out,
                       cudaStream_t s);
}  // namespace vx

extern "C" {

int vx_abi_version(void) { return VX_ABI_VERSION; }
const char* vx_last_error(void) { return g_err; }
int64_t vx_launch_count(void) { return g_launches.load(); }

int vx_voxel_keys(const double* d_xyz, int64_t n, double voxel_size, int64_t* d_keys, void* stream) {
    if (!(voxel_size > 0)) {
        set_error("voxel_size must be positive");
        return VX_E_INPUT;
    }
    if (n <= 0) return VX_OK;
    cudaStream_t s = as_stream(stream);
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    Scratch& sc = scratch();
    VX_TRY(sc.a.reserve(sizeof(int), s));
    if (!sc.host) VX_CUDA(cudaMallocHost(&sc.host, 256));
    VX_CUDA(cudaMemsetAsync(sc.a.ptr, 0, sizeof(int), s));
    k_voxel_keys<<<unsigned((n * 3 + 255) / 256), 256, 0, s>>>(d_xyz, n, voxel_size, d_keys,
                                                               sc.a.as<int>());
    count_launch();
    VX_CHECK_LAUNCH();
    VX_CUDA(cudaMemcpyAsync(sc.host, sc.a.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaStreamSynchronize(s));
    if (sc.host[0] & 1) {
        set_error("cannot hash non-finite positions");
        return VX_E_INPUT;
    }
    if (sc.host[0] & 2) {
        set_error("voxel key overflows int64");
        return VX_E_RANGE;
    }
    return VX_OK;
}

int vx_kernel_matrix(const double* d_xa, int64_t na, const double* d_xb, int64_t nb, double lam,
                     int32_t kernel, double* d_out, void* stream) {
    if (!(lam > 0)) {
        set_error("kernel constant must be positive");
        return VX_E_INPUT;
    }
    if (na <= 0 || nb <= 0) return VX_OK;
    cudaStream_t s = as_stream(stream);
    k_kernel_matrix<<<unsigned((na * nb + 255) / 256), 256, 0, s>>>(d_xa, na, d_xb, nb, lam, kernel,
                                                                    d_out);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

int vx_mesh_grid(const double* d_ext, int64_t num, int32_t n_s, int32_t n_r, double* d_out,
                 void* stream) {
    if (n_s < 1 || n_r < 1) {
        set_error("n_s and n_r must be at least 1");
        return VX_E_INPUT;
    }
    if (num <= 0) return VX_OK;
    const int64_t tot = num * int64_t(n_s * n_r) * (n_s * n_r);
    cudaStream_t s = as_stream(stream);
    k_mesh_grid<<<unsigned((tot + 255) / 256), 256, 0, s>>>(d_ext, num, n_s, n_r, d_out);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

int vx_select_axis_batch(const double* d_points, const int64_t* d_offsets, int64_t num, int8_t* d_axis,
                         void* stream) {
    if (num <= 0) return VX_OK;
    cudaStream_t s = as_stream(stream);
    k_select_axis<<<unsigned((num + 127) / 128), 128, 0, s>>>(d_points, d_offsets, num, d_axis);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

int vx_gpr_solve_batch(const VxGprBatch* b, void* stream) {
    if (!b) {
        set_error("null batch");
        return VX_E_INPUT;
    }
    const int64_t P = b->num_problems;
    if (P <= 0) return VX_OK;
    if (b->d_full && !b->d_full_off) {
        set_error("d_full requires d_full_off");
        return VX_E_INPUT;
    }
    cudaStream_t s = as_stream(stream);
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    Scratch& sc = scratch();
    if (!sc.host) VX_CUDA(cudaMallocHost(&sc.host, 256));
    VX_TRY(sc.a.reserve(size_t(P) * 4, s));
    VX_TRY(sc.b.reserve(256, s));
    int* cnt = sc.b.as<int>();
    VX_CUDA(cudaMemsetAsync(cnt, 0, 256, s));   // [0,16) counts, [16,32) fill, [32,48) bases
    const unsigned g = unsigned((P + 255) / 256);
    k_problem_count<<<g, 256, 0, s>>>(b->d_x_off, P, cnt);
    count_launch();
    VX_CUDA(cudaMemcpyAsync(sc.host, cnt, NUM_BUCKETS * sizeof(int), cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaStreamSynchronize(s));
    int counts[NUM_BUCKETS];
    int64_t offs[NUM_BUCKETS];
    int64_t acc = 0;
    for (int k = 0; k < NUM_BUCKETS; ++k) {
        counts[k] = sc.host[k];
        offs[k] = acc;
        sc.host[32 + k] = int(acc);
        acc += counts[k];
    }
    VX_CUDA(cudaMemcpyAsync(cnt + 32, sc.host + 32, NUM_BUCKETS * sizeof(int), cudaMemcpyHostToDevice, s));
    k_problem_buckets<<<g, 256, 0, s>>>(b->d_x_off, P, sc.a.as<int32_t>(), cnt + 16, cnt + 32);
    count_launch();
    VX_CHECK_LAUNCH();
    for (int k = NUM_BUCKETS - 1; k >= 0; --k) {
        if (counts[k] == 0) continue;
        VX_TRY(launch_problem_solve(*b, sc.a.as<int32_t>() + offs[k], counts[k], b->max_n, b->max_m,
                                    sc.c, s, k));
    }
    // the scratch item list must outlive the kernels
    VX_CUDA(cudaStreamSynchronize(s));
    return VX_OK;
}

int vx_subgrid_moments(const double* d_points, const double* d_weights, int64_t num, int32_t k,
                       const double* d_center, double* d_pos, double* d_phi, void* stream) {
    if (k < 1) {
        set_error("subgrid needs at least one point");
        return VX_E_INPUT;
    }
    return launch_moments(d_points, d_weights, num, k, d_center, d_pos, d_phi, as_stream(stream));
}

int vx_gaussians_from_predictions(const double* d_pred_xyz, const double* d_pred_rgb,
                                  const double* d_pred_var, const int64_t* d_keys, int64_t count,
                                  int64_t points_per_prediction, const VxCamera* camera,
                                  const double* d_image, const VxSplatConfig* cfg, VxGaussianOut* out,
                                  void* stream) {
    if (!camera || !cfg || !out) {
        set_error("camera, cfg and out are required");
        return VX_E_INPUT;
    }
    return launch_gaussians(d_pred_xyz, d_pred_rgb, d_pred_var, nullptr, nullptr, nullptr, d_keys,
                            count, int(points_per_prediction), *camera, d_image, *cfg, *out,
                            as_stream(stream));
}

int vx_map_create(const VxMapConfig* cfg, VxMap** out) {
    if (!cfg || !out) {
        set_error("null argument");
        return VX_E_INPUT;
    }
    if (!(cfg->voxel_size > 0)) {
        set_error("voxel_size must be positive");
        return VX_E_INPUT;
    }
    if (!(cfg->sensor_var >= 0)) {
        set_error("sensor_var must be nonnegative");
        return VX_E_INPUT;
    }
    if (cfg->n_s < 1 || cfg->n_r < 1 || cfg->n_s * cfg->n_r > 16) {
        set_error("n_s, n_r must be >= 1 with n_s * n_r <= 16");
        return VX_E_INPUT;
    }
    if (!(cfg->kernel_lambda > 0)) {
        set_error("kernel constant must be positive");
        return VX_E_INPUT;
    }
    if (cfg->shard_world < 1 || cfg->shard_rank < 0 || cfg->shard_rank >= cfg->shard_world) {
        set_error("bad shard (rank %d, world %d)", cfg->shard_rank, cfg->shard_world);
        return VX_E_INPUT;
    }
    int rc = VX_OK;
    VxMap* m = map_new(*cfg, &rc);
    if (!m) return rc;
    *out = m;
    return VX_OK;
}

int vx_map_destroy(VxMap* map) {
    if (map) map_delete(map);
    return VX_OK;
}

int vx_map_clear(VxMap* map, void* stream) {
    if (!map) {
        set_error("null map");
        return VX_E_INPUT;
    }
    return map_clear(map, as_stream(stream));
}

int vx_map_view(VxMap* map, VxMapView* out) {
    if (!map || !out) {
        set_error("null argument");
        return VX_E_INPUT;
    }
    map_fill_view(map, out);
    return VX_OK;
}

int vx_map_store_frame(VxMap* map, const double* d_xyz, const double* d_rgb, int64_t n,
                       VxFrameInfo* info, void* stream) {
    if (!map) {
        set_error("null map");
        return VX_E_INPUT;
    }
    return map_store_frame(map, d_xyz, d_rgb, n, info, as_stream(stream));
}

int vx_map_partition_by_owner(VxMap* map, const double* d_xyz, const double* d_rgb, int64_t n,
                              int64_t global_base, double* d_out_xyz, double* d_out_rgb,
                              int64_t* d_out_index, int64_t* h_counts, void* stream) {
    if (!map || !h_counts || (n > 0 && (!d_xyz || !d_rgb || !d_out_xyz || !d_out_rgb || !d_out_index))) {
        set_error("null argument");
        return VX_E_INPUT;
    }
    return map_partition_by_owner(map, d_xyz, d_rgb, n, global_base, d_out_xyz, d_out_rgb,
                                  d_out_index, h_counts, as_stream(stream));
}

int vx_map_densify(VxMap* map, VxDensifyInfo* info, void* stream) {
    if (!map) {
        set_error("null map");
        return VX_E_INPUT;
    }
    return map_densify(map, info, as_stream(stream));
}

int vx_map_init_gaussians(VxMap* map, const int32_t* d_voxels, int64_t count, const VxCamera* camera,
                          const double* d_image, const VxSplatConfig* cfg, VxGaussianOut* out,
                          void* stream) {
    if (!map || !camera || !cfg || !out) {
        set_error("null argument");
        return VX_E_INPUT;
    }
    return map_init_gaussians(map, d_voxels, count, *camera, d_image, *cfg, *out, as_stream(stream));
}

int vx_map_ingest(VxMap* map, const double* d_xyz, const double* d_rgb, int64_t n,
                  const VxCamera* camera, const double* d_image, const VxSplatConfig* cfg,
                  VxGaussianOut* out, int64_t out_capacity, int64_t* out_records,
                  VxFrameInfo* frame_info, VxDensifyInfo* densify_info, void* stream) {
    if (!map) {
        set_error("null map");
        return VX_E_INPUT;
    }
    if (camera && !cfg) {
        set_error("camera requires a splat config");
        return VX_E_INPUT;
    }
    return map_ingest(map, d_xyz, d_rgb, n, camera, d_image, cfg, out, out_capacity, out_records,
                      frame_info, densify_info, as_stream(stream));
}

int vx_map_emit_first_gaussians(VxMap* map, const VxCamera* camera, const double* d_image,
                                const VxSplatConfig* cfg, VxGaussianOut* out,
                                int64_t out_capacity, int64_t* out_records, void* stream) {
    if (!map || !camera || !cfg || !out) {
        set_error("null argument");
        return VX_E_INPUT;
    }
    return map_emit_first_gaussians(map, camera, d_image, cfg, out, out_capacity, out_records,
                                    as_stream(stream));
}

int vx_map_lookup(VxMap* map, const int64_t* d_keys, int64_t n, int32_t* d_voxels, void* stream) {
    if (!map) {
        set_error("null map");
        return VX_E_INPUT;
    }
    return map_lookup(map, d_keys, n, d_voxels, as_stream(stream));
}

int vx_map_set_frame_keys(VxMap* map, const int64_t* d_keys, int64_t n, void* stream) {
    if (!map) {
        set_error("null map");
        return VX_E_INPUT;
    }
    return map_set_frame_keys(map, d_keys, n, as_stream(stream));
}

int vx_map_apply_prediction(VxMap* map, const int64_t* h_key, const double* d_xyz, const double* d_rgb,
                            const double* d_var, int64_t m, uint8_t* h_before_after, void* stream) {
    if (!map || !h_key || !h_before_after) {
        set_error("null argument");
        return VX_E_INPUT;
    }
    return map_apply_prediction(map, h_key, d_xyz, d_rgb, d_var, m, h_before_after, as_stream(stream));
}

int vx_map_configure_solver(VxMap* map, int32_t n_s, int32_t n_r, double kernel_lambda, double jitter,
                            int32_t kernel) {
    if (!map) {
        set_error("null map");
        return VX_E_INPUT;
    }
    return map_configure_solver(map, n_s, n_r, kernel_lambda, jitter, kernel);
}

int vx_init_color(const double* d_positions, const double* d_fallback, int64_t n, const VxCamera* camera,
                  const double* d_image, double* d_sh0, void* stream) {
    if (!camera) {
        set_error("camera required");
        return VX_E_INPUT;
    }
    return launch_init_color(d_positions, d_fallback, n, *camera, d_image, d_sh0, as_stream(stream));
}

int vx_project_points(const double* d_pos, const double* d_scale, const double* d_rot, int64_t n,
                      const VxCamera* camera, double near_plane, double* d_mean2d, double* d_cov2d,
                      double* d_depth, double* d_radius, uint8_t* d_valid, int64_t* d_bbox,
                      void* stream) {
    if (!camera || n < 0) {
        set_error("project_points: camera required, n >= 0");
        return VX_E_INPUT;
    }
    return project_points(d_pos, d_scale, d_rot, n, *camera, near_plane, d_mean2d, d_cov2d, d_depth,
                          d_radius, d_valid, d_bbox, as_stream(stream));
}

int vx_render(const double* d_pos, const double* d_scale, const double* d_rot, const double* d_opacity,
              const double* d_sh0, int64_t n, const VxCamera* camera, double near_plane,
              double* d_color, double* d_depth, double* d_silhouette, void* stream) {
    if (!camera || n < 0 || camera->width <= 0 || camera->height <= 0) {
        set_error("render: camera with a positive image size required, n >= 0");
        return VX_E_INPUT;
    }
    return render_splats(d_pos, d_scale, d_rot, d_opacity, d_sh0, n, *camera, near_plane, d_color,
                         d_depth, d_silhouette, as_stream(stream));
}

int vx_profile(int enable) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    prof_collect();
    for (int k = 0; k < P_COUNT; ++k) {
        g_prof.ms[k] = 0;
        g_prof.n[k] = 0;
    }
    g_prof.on = enable != 0;
    return VX_OK;
}

int vx_profile_read(double* ms, int64_t* launches, int32_t max_stages) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    prof_collect();
    for (int k = 0; k < P_COUNT && k < max_stages; ++k) {
        ms[k] = g_prof.ms[k];
        launches[k] = g_prof.n[k];
    }
    return P_COUNT;
}

int vx_decode_ply(const void* d_records, int64_t n, double* d_xyz, double* d_rgb, void* stream) {
    if (n > 0 && (!d_records || !d_xyz || !d_rgb)) {
        set_error("null argument");
        return VX_E_INPUT;
    }
    return launch_decode_ply(static_cast<const uint8_t*>(d_records), n, d_xyz, d_rgb,
                             as_stream(stream));
}

int vx_pack_map_records(const VxGaussianOut* records, int64_t count, void* d_out, void* stream) {
    if (!records || (!d_out && count > 0)) {
        set_error("null argument");
        return VX_E_INPUT;
    }
    return launch_pack_records(*records, count, d_out, as_stream(stream));
}

int vx_fp64_peak(double* tflops, void* stream) {
    // max of the DFMA pipe and the DMMA (FP64 tensor) pipe, which share one
    // FP64 datapath (tools/dmma_peak.cu); both timed on all SMs
    cudaStream_t s = as_stream(stream);
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    Scratch& sc = scratch();
    VX_TRY(sc.a.reserve(64, s));
    const int blocks = sm_count() * 8, iters = 4096;
    cudaEvent_t e0, e1;
    VX_CUDA(cudaEventCreate(&e0));
    VX_CUDA(cudaEventCreate(&e1));
    double best_tf = 0.0;
    for (int kind = 0; kind < 2; ++kind) {
        auto launch = [&]() {
            if (kind == 0) k_dfma_peak<<<blocks, 256, 0, s>>>(sc.a.as<double>(), iters, 0.999999, 1e-7);
            else k_dmma_peak<<<blocks, 256, 0, s>>>(sc.a.as<double>(), iters / 8, 0.999999, 1e-7);
            count_launch();
        };
        launch();   // warm-up
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            VX_CUDA(cudaEventRecord(e0, s));
            launch();
            VX_CUDA(cudaEventRecord(e1, s));
            VX_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            VX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        // DFMA: 2 flops x 8 chains per thread-iteration; DMMA: 8x8x4 x 2 flops
        // per warp-instruction, 8 chains, iters/8 iterations
        const double flops = kind == 0 ? 2.0 * 8.0 * double(iters) * double(blocks) * 256.0
                                       : 512.0 * 8.0 * double(iters / 8) * double(blocks) * 8.0;
        const double tf = flops / (double(best) * 1e-3) / 1e12;
        if (tf > best_tf) best_tf = tf;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tflops = best_tf;
    return VX_OK;
}

}  // extern "C"
