// Tile-based forward splat rasteriser (renderer.py:90-207):
// the consumer of the Gaussian records the mapping path produces (SURVEY
// §8(f) row 4).
//
//   k_project        thread per primitive: camera transform, 2D covariance
//                    J W Phi W^T J^T + dilation (renderer.py:99-124), 3-sigma
//                    radius, pixel bbox, validity (125-137); tile count
//   depth order      stable LSD radix sort of the valid primitives by the
//                    bits of their (positive) depth, low word then high word:
//                    front to back, ties by index (depth_order, 176-179)
//   tile binning     every ranked primitive emits (tile, rank) for each
//                    16x16 tile its bbox touches; a stable sort by tile keeps
//                    each tile's list in global front-to-back order
//   k_render_tiles   CTA per tile, thread per pixel: the tile's primitives are
//                    staged through shared memory 256 at a time and blended in
//                    order exactly as render() (184-207) updates a pixel:
//                    alpha = min(0.99, o exp(power)), skipped below 1/255,
//                    live while T >= 1e-4; the CTA stops once every pixel of
//                    the tile is dead (a dead pixel never changes again)
//
// FP64 throughout; the per-pixel quadratic form and the blend use the
// reference's NumPy operation order without FMA contraction, so a pixel's
// value differs from the reference only through exp() (<= 1 ulp) and the
// covariance's 3x3 products (einsum order).
#include <cmath>
#include <mutex>

#include "vx_common.cuh"
#include "vx_internal.h"

namespace vx {

constexpr int RT = 16;                          // tile edge (pixels)
constexpr int RT2 = RT * RT;
constexpr double ALPHA_CEILING = 0.99;          // renderer.py:27
constexpr double ALPHA_SKIP = 1.0 / 255.0;      // renderer.py:28
constexpr double TRANSMITTANCE_EPS = 1e-4;      // renderer.py:29
constexpr double COV_DILATION = 0.3;            // renderer.py:30
constexpr double RADIUS_SIGMAS = 3.0;           // renderer.py:31
constexpr double SH0_C0 = 0.28209479177;        // splat_init.py:22

struct ProjOut {
    double* mean2d;     // (n,2)
    double* cov2d;      // (n,4) row-major 2x2 (symmetrised, dilated)
    double* depth;      // (n)
    double* radius;     // (n)
    uint8_t* valid;     // (n)
    int64_t* bbox;      // (n,4) x0, x1, y0, y1 (half-open), zero when invalid
    int32_t* ntiles;    // (n) tiles touched (render only) or null
};

__global__ void k_project(const double* __restrict__ pos, const double* __restrict__ scale,
                          const double* __restrict__ rot, int64_t n, VxCamera cam, double near,
                          ProjOut o) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double px = pos[i * 3], py = pos[i * 3 + 1], pz = pos[i * 3 + 2];
    const double* R = cam.R;
    // pts @ R^T + t (camera.py:52-54)
    const double x = xadd(xadd(xadd(xmul(px, R[0]), xmul(py, R[1])), xmul(pz, R[2])), cam.t[0]);
    const double y = xadd(xadd(xadd(xmul(px, R[3]), xmul(py, R[4])), xmul(pz, R[5])), cam.t[1]);
    const double z = xadd(xadd(xadd(xmul(px, R[6]), xmul(py, R[7])), xmul(pz, R[8])), cam.t[2]);
    bool valid = z > near;
    const double zs = valid ? z : 1.0;
    const double u = xadd(xdiv(xmul(cam.fx, x), zs), cam.cx);
    const double v = xadd(xdiv(xmul(cam.fy, y), zs), cam.cy);
    // quaternion (w,x,y,z) -> rotation, normalised (geometry.py:34-48)
    double qw = rot[i * 4], qx = rot[i * 4 + 1], qy = rot[i * 4 + 2], qz = rot[i * 4 + 3];
    const double qn = sqrt(xadd(xadd(xadd(xmul(qw, qw), xmul(qx, qx)), xmul(qy, qy)), xmul(qz, qz)));
    qw = xdiv(qw, qn); qx = xdiv(qx, qn); qy = xdiv(qy, qn); qz = xdiv(qz, qn);
    double G[9];
    G[0] = 1 - 2 * (qy * qy + qz * qz); G[1] = 2 * (qx * qy - qw * qz); G[2] = 2 * (qx * qz + qw * qy);
    G[3] = 2 * (qx * qy + qw * qz); G[4] = 1 - 2 * (qx * qx + qz * qz); G[5] = 2 * (qy * qz - qw * qx);
    G[6] = 2 * (qx * qz - qw * qy); G[7] = 2 * (qy * qz + qw * qx); G[8] = 1 - 2 * (qx * qx + qy * qy);
    // Phi = G diag(S^2) G^T, M = W Phi W^T (W = camera rotation)
    double s2[3];
    for (int k = 0; k < 3; ++k) s2[k] = scale[i * 3 + k] * scale[i * 3 + k];
    double phi[9];
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j) acc += G[a * 3 + j] * s2[j] * G[c * 3 + j];
            phi[a * 3 + c] = acc;
        }
    double tmp[9], M[9];
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j) acc += R[a * 3 + j] * phi[j * 3 + c];
            tmp[a * 3 + c] = acc;
        }
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j) acc += tmp[a * 3 + j] * R[c * 3 + j];
            M[a * 3 + c] = acc;
        }
    // perspective Jacobian at the mean (renderer.py:115-119)
    const double J00 = cam.fx / zs, J02 = -cam.fx * x / (zs * zs);
    const double J11 = cam.fy / zs, J12 = -cam.fy * y / (zs * zs);
    // cov2d = J M J^T
    const double JM0[3] = {J00 * M[0] + J02 * M[6], J00 * M[1] + J02 * M[7], J00 * M[2] + J02 * M[8]};
    const double JM1[3] = {J11 * M[3] + J12 * M[6], J11 * M[4] + J12 * M[7], J11 * M[5] + J12 * M[8]};
    double c00 = JM0[0] * J00 + JM0[2] * J02;
    double c01 = JM0[1] * J11 + JM0[2] * J12;
    double c10 = JM1[0] * J00 + JM1[2] * J02;
    double c11 = JM1[1] * J11 + JM1[2] * J12;
    c00 = xadd(c00, COV_DILATION);
    c11 = xadd(c11, COV_DILATION);
    const double b = xmul(0.5, xadd(c01, c10));         // 0.5 (cov + cov^T)
    const double a = xmul(0.5, xadd(c00, c00)), c = xmul(0.5, xadd(c11, c11));
    // largest eigenvalue, 3-sigma radius (renderer.py:125-129)
    const double mid = xmul(0.5, xadd(a, c));
    const double h = xmul(0.5, xsub(a, c));
    double dq = xadd(xmul(h, h), xmul(b, b));
    const double disc = sqrt(dq > 0.0 ? dq : 0.0);
    const double lam = xadd(mid, disc);
    const double radius = xmul(RADIUS_SIGMAS, sqrt(lam > 0.0 ? lam : 0.0));
    const bool on_image = xadd(u, radius) >= 0.0 && xsub(u, radius) <= double(cam.width - 1) &&
                          xadd(v, radius) >= 0.0 && xsub(v, radius) <= double(cam.height - 1);
    valid = valid && on_image && isfinite(u) && isfinite(v);
    auto clampd = [](double t, double hi) { return t < 0.0 ? 0.0 : (t > hi ? hi : t); };
    const int64_t x0 = int64_t(clampd(ceil(xsub(u, radius)), double(cam.width)));
    const int64_t x1 = int64_t(clampd(xadd(floor(xadd(u, radius)), 1.0), double(cam.width)));
    const int64_t y0 = int64_t(clampd(ceil(xsub(v, radius)), double(cam.height)));
    const int64_t y1 = int64_t(clampd(xadd(floor(xadd(v, radius)), 1.0), double(cam.height)));
    valid = valid && x1 > x0 && y1 > y0;
    o.mean2d[i * 2] = u;
    o.mean2d[i * 2 + 1] = v;
    o.cov2d[i * 4] = a;
    o.cov2d[i * 4 + 1] = b;
    o.cov2d[i * 4 + 2] = b;
    o.cov2d[i * 4 + 3] = c;
    o.depth[i] = z;
    o.radius[i] = radius;
    o.valid[i] = valid ? 1 : 0;
    o.bbox[i * 4] = valid ? x0 : 0;
    o.bbox[i * 4 + 1] = valid ? x1 : 0;
    o.bbox[i * 4 + 2] = valid ? y0 : 0;
    o.bbox[i * 4 + 3] = valid ? y1 : 0;
    if (o.ntiles) {
        int32_t t = 0;
        if (valid) t = int32_t(((x1 - 1) / RT - x0 / RT + 1) * ((y1 - 1) / RT - y0 / RT + 1));
        o.ntiles[i] = t;
    }
}

// ---------------------------------------------------------------- ordering
__global__ void k_valid_flags(const uint8_t* valid, int64_t n, int32_t* flags) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = valid[i];
}

// valid primitive -> compact slot: low and high words of its depth bits
// (positive doubles order like their bit patterns), value = primitive index
__global__ void k_depth_keys(const uint8_t* valid, const int32_t* scan, const double* depth,
                             int64_t n, uint32_t* klo, uint32_t* khi, uint32_t* idx) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || !valid[i]) return;
    const int32_t s = scan[i];
    const uint64_t b = uint64_t(__double_as_longlong(depth[i]));
    klo[s] = uint32_t(b);
    khi[s] = uint32_t(b >> 32);
    idx[s] = uint32_t(i);
}

__global__ void k_gather_u32(const uint32_t* src, const uint32_t* perm, int64_t m, uint32_t* dst) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < m) dst[r] = src[perm[r]];
}

// ranked primitive r (front to back) -> its tile count
__global__ void k_rank_tiles(const uint32_t* order, int64_t m, const int32_t* ntiles, int32_t* cnt) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < m) cnt[r] = ntiles[order[r]];
}

__global__ void k_emit_tiles(const uint32_t* order, int64_t m, const int64_t* bbox, const int32_t* off,
                             int tiles_x, uint32_t* tkey, uint32_t* tval) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int64_t g = order[r];
    const int tx0 = int(bbox[g * 4] / RT), tx1 = int((bbox[g * 4 + 1] - 1) / RT);
    const int ty0 = int(bbox[g * 4 + 2] / RT), ty1 = int((bbox[g * 4 + 3] - 1) / RT);
    int32_t o = off[r];
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            tkey[o] = uint32_t(ty * tiles_x + tx);
            tval[o] = uint32_t(r);
            ++o;
        }
}

__global__ void k_tile_ranges(const uint32_t* tkey, int64_t e, int32_t* tstart, int32_t* tend) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= e) return;
    const uint32_t k = tkey[j];
    if (j == 0 || tkey[j - 1] != k) tstart[k] = int32_t(j);
    if (j == e - 1 || tkey[j + 1] != k) tend[k] = int32_t(j + 1);
}

struct RenderArgs {
    const double* mean2d;
    const double* cov2d;
    const double* depth;
    const int64_t* bbox;
    const double* opacity;
    const double* sh0;
    const uint32_t* order;      // rank -> primitive
    const uint32_t* tval;       // tile-sorted ranks
    const int32_t* tstart;
    const int32_t* tend;
    int width, height, tiles_x;
    double* color;
    double* dep;
    double* sil;
};

// CTA per 16x16 tile, thread per pixel (render(), renderer.py:184-207)
__global__ void __launch_bounds__(RT2) k_render_tiles(RenderArgs a) {
    __shared__ double s_m0[RT2], s_m1[RT2], s_a[RT2], s_b[RT2], s_c[RT2], s_det[RT2], s_op[RT2],
        s_z[RT2], s_rgb[RT2 * 3];
    __shared__ int s_box[RT2 * 4];
    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int px = tx * RT + (threadIdx.x % RT), py = ty * RT + (threadIdx.x / RT);
    const bool inside = px < a.width && py < a.height;
    double cr = 0.0, cg = 0.0, cb = 0.0, dd = 0.0, ss = 0.0, T = 1.0;
    const int beg = a.tstart[tile], end = a.tend[tile];
    for (int c0 = beg; c0 < end; c0 += RT2) {
        // stop when no pixel of the tile can change any more
        const bool alive = inside && T >= TRANSMITTANCE_EPS;
        if (__syncthreads_or(alive) == 0) break;
        const int j = c0 + threadIdx.x;
        if (j < end) {
            const int64_t g = a.order[a.tval[j]];
            const double A = a.cov2d[g * 4], B = a.cov2d[g * 4 + 1], C = a.cov2d[g * 4 + 3];
            s_m0[threadIdx.x] = a.mean2d[g * 2];
            s_m1[threadIdx.x] = a.mean2d[g * 2 + 1];
            s_a[threadIdx.x] = A;
            s_b[threadIdx.x] = B;
            s_c[threadIdx.x] = C;
            s_det[threadIdx.x] = xsub(xmul(A, C), xmul(B, B));   // gaussian_patch, renderer.py:155
            s_op[threadIdx.x] = a.opacity[g];
            s_z[threadIdx.x] = a.depth[g];
            for (int k = 0; k < 3; ++k)      // sh0_to_rgb (splat_init.py:32-34)
                s_rgb[threadIdx.x * 3 + k] = xadd(xmul(a.sh0[g * 3 + k], SH0_C0), 0.5);
            for (int k = 0; k < 4; ++k) s_box[threadIdx.x * 4 + k] = int(a.bbox[g * 4 + k]);
        }
        __syncthreads();
        const int cnt = end - c0 < RT2 ? end - c0 : RT2;
        if (inside) {
            const double fx = double(px), fy = double(py);
            for (int k = 0; k < cnt; ++k) {
                if (px < s_box[k * 4] || px >= s_box[k * 4 + 1] || py < s_box[k * 4 + 2] ||
                    py >= s_box[k * 4 + 3])
                    continue;
                // power = -0.5 (c dx^2 - 2 b dx dy + a dy^2) / det (renderer.py:151-157)
                const double dx = xsub(fx, s_m0[k]), dy = xsub(fy, s_m1[k]);
                const double t1 = xmul(s_c[k], xmul(dx, dx));
                const double t2 = xmul(xmul(xmul(2.0, s_b[k]), dx), dy);
                const double t3 = xmul(s_a[k], xmul(dy, dy));
                const double power = xdiv(xmul(-0.5, xadd(xsub(t1, t2), t3)), s_det[k]);
                // alpha_patch (renderer.py:160-173)
                double alpha = xmul(s_op[k], exp(power));
                alpha = alpha < ALPHA_CEILING ? alpha : ALPHA_CEILING;
                if (alpha < ALPHA_SKIP) alpha = 0.0;
                if (T >= TRANSMITTANCE_EPS) {
                    const double w = xmul(alpha, T);
                    cr = xadd(cr, xmul(w, s_rgb[k * 3]));
                    cg = xadd(cg, xmul(w, s_rgb[k * 3 + 1]));
                    cb = xadd(cb, xmul(w, s_rgb[k * 3 + 2]));
                    dd = xadd(dd, xmul(w, s_z[k]));
                    ss = xadd(ss, w);
                    T = xmul(T, xsub(1.0, alpha));
                }
            }
        }
        __syncthreads();
    }
    if (inside) {
        const int64_t p = int64_t(py) * a.width + px;
        a.color[p * 3] = cr;
        a.color[p * 3 + 1] = cg;
        a.color[p * 3 + 2] = cb;
        a.dep[p] = dd;
        a.sil[p] = ss;
    }
}

// ---------------------------------------------------------------- host
namespace {
struct RenderScratch {
    DevBuf mean2d, cov2d, depth, radius, valid, bbox, ntiles, flags, scan, klo, khi, idx, klo2, khi2,
        idx2, order, cnt, off, tkey, tval, tkey2, tval2, tstart, tend, tmp, sort_tmp;
};
RenderScratch g_rs;          // process-wide scratch, grown on demand
std::mutex g_rs_mu;          // one render at a time per process (host threads)
cudaEvent_t g_rs_done = nullptr;   // last render's kernels: a render on another
                                   // stream waits for them before reusing scratch
}  // namespace

int launch_project(const double* pos, const double* scale, const double* rot, int64_t n,
                   const VxCamera& cam, double near, const ProjOut& o, cudaStream_t s) {
    if (n <= 0) return VX_OK;
    k_project<<<unsigned((n + 127) / 128), 128, 0, s>>>(pos, scale, rot, n, cam, near, o);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

int project_points(const double* pos, const double* scale, const double* rot, int64_t n,
                   const VxCamera& cam, double near, double* mean2d, double* cov2d, double* depth,
                   double* radius, uint8_t* valid, int64_t* bbox, cudaStream_t s) {
    ProjOut o{mean2d, cov2d, depth, radius, valid, bbox, nullptr};
    return launch_project(pos, scale, rot, n, cam, near, o, s);
}

static int render_splats_impl(const double* pos, const double* scale, const double* rot,
                              const double* opacity, const double* sh0, int64_t n,
                              const VxCamera& cam, double near, double* color, double* depth,
                              double* sil, cudaStream_t s);

int render_splats(const double* pos, const double* scale, const double* rot, const double* opacity,
                  const double* sh0, int64_t n, const VxCamera& cam, double near, double* color,
                  double* depth, double* sil, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_rs_mu);
    if (g_rs_done == nullptr) VX_CUDA(cudaEventCreateWithFlags(&g_rs_done, cudaEventDisableTiming));
    VX_CUDA(cudaStreamWaitEvent(s, g_rs_done, 0));
    const int rc = render_splats_impl(pos, scale, rot, opacity, sh0, n, cam, near, color, depth, sil, s);
    VX_CUDA(cudaEventRecord(g_rs_done, s));
    return rc;
}

static int render_splats_impl(const double* pos, const double* scale, const double* rot,
                              const double* opacity, const double* sh0, int64_t n,
                              const VxCamera& cam, double near, double* color, double* depth,
                              double* sil, cudaStream_t s) {
    const int W = cam.width, H = cam.height;
    const int tiles_x = (W + RT - 1) / RT, tiles_y = (H + RT - 1) / RT;
    const int ntl = tiles_x * tiles_y;
    RenderScratch& r = g_rs;
    if (n >= (int64_t(1) << 31) - 1) {
        set_error("render: %lld primitives exceed the 2^31 limit", (long long)n);
        return VX_E_INPUT;
    }
    VX_TRY(r.tstart.reserve(size_t(ntl) * 4, s));
    VX_TRY(r.tend.reserve(size_t(ntl) * 4, s));
    VX_CUDA(cudaMemsetAsync(r.tstart.ptr, 0, size_t(ntl) * 4, s));
    VX_CUDA(cudaMemsetAsync(r.tend.ptr, 0, size_t(ntl) * 4, s));
    int64_t m = 0;
    int64_t e = 0;
    if (n > 0) {
        VX_TRY(r.mean2d.reserve(size_t(n) * 16, s));
        VX_TRY(r.cov2d.reserve(size_t(n) * 32, s));
        VX_TRY(r.depth.reserve(size_t(n) * 8, s));
        VX_TRY(r.radius.reserve(size_t(n) * 8, s));
        VX_TRY(r.valid.reserve(size_t(n), s));
        VX_TRY(r.bbox.reserve(size_t(n) * 32, s));
        VX_TRY(r.ntiles.reserve(size_t(n) * 4, s));
        VX_TRY(r.flags.reserve(size_t(n) * 4, s));
        VX_TRY(r.scan.reserve(size_t(n) * 4 + 8, s));
        ProjOut o{r.mean2d.as<double>(), r.cov2d.as<double>(), r.depth.as<double>(),
                  r.radius.as<double>(), r.valid.as<uint8_t>(), r.bbox.as<int64_t>(),
                  r.ntiles.as<int32_t>()};
        VX_TRY(launch_project(pos, scale, rot, n, cam, near, o, s));
        const unsigned nb = unsigned((n + 255) / 256);
        k_valid_flags<<<nb, 256, 0, s>>>(r.valid.as<uint8_t>(), n, r.flags.as<int32_t>());
        count_launch();
        int32_t* d_m = r.scan.as<int32_t>() + n;
        VX_TRY(scan_exclusive_i32(r.flags.as<int32_t>(), r.scan.as<int32_t>(), n, d_m, r.tmp, s));
        int32_t hm = 0;
        VX_CUDA(cudaMemcpyAsync(&hm, d_m, 4, cudaMemcpyDeviceToHost, s));
        VX_CUDA(cudaStreamSynchronize(s));
        m = hm;
    }
    if (m > 0) {
        for (DevBuf* b : {&r.klo, &r.khi, &r.idx, &r.klo2, &r.khi2, &r.idx2, &r.order})
            VX_TRY(b->reserve(size_t(m) * 4, s));
        VX_TRY(r.cnt.reserve(size_t(m) * 4, s));
        VX_TRY(r.off.reserve(size_t(m) * 4 + 8, s));
        k_depth_keys<<<unsigned((n + 255) / 256), 256, 0, s>>>(
            r.valid.as<uint8_t>(), r.scan.as<int32_t>(), r.depth.as<double>(), n, r.klo.as<uint32_t>(),
            r.khi.as<uint32_t>(), r.idx.as<uint32_t>());
        count_launch();
        const unsigned mb = unsigned((m + 255) / 256);
        // stable LSD over the 64-bit depth of the compact slots (slot order =
        // primitive order): low words first, then the high words gathered in
        // that order; slot -> primitive (idx) at the end
        uint32_t* va = r.idx2.as<uint32_t>();
        uint32_t* vb = r.order.as<uint32_t>();
        bool alt = false;
        VX_TRY(radix_sort_pairs(r.klo.as<uint32_t>(), va, r.klo2.as<uint32_t>(), vb, m, 32, r.sort_tmp,
                                s, &alt, /*vals_identity=*/true));
        uint32_t* perm1 = alt ? vb : va;
        uint32_t* other = alt ? va : vb;
        k_gather_u32<<<mb, 256, 0, s>>>(r.khi.as<uint32_t>(), perm1, m, r.khi2.as<uint32_t>());
        count_launch();
        VX_CHECK_LAUNCH();
        bool alt2 = false;
        VX_TRY(radix_sort_pairs(r.khi2.as<uint32_t>(), perm1, r.khi.as<uint32_t>(), other, m, 32,
                                r.sort_tmp, s, &alt2));
        const uint32_t* slots = alt2 ? other : perm1;
        uint32_t* order = r.klo.as<uint32_t>();
        k_gather_u32<<<mb, 256, 0, s>>>(r.idx.as<uint32_t>(), slots, m, order);
        count_launch();
        VX_CHECK_LAUNCH();
        k_rank_tiles<<<mb, 256, 0, s>>>(order, m, r.ntiles.as<int32_t>(), r.cnt.as<int32_t>());
        count_launch();
        int32_t* d_e = r.off.as<int32_t>() + m;
        VX_TRY(scan_exclusive_i32(r.cnt.as<int32_t>(), r.off.as<int32_t>(), m, d_e, r.tmp, s));
        int32_t he = 0;
        VX_CUDA(cudaMemcpyAsync(&he, d_e, 4, cudaMemcpyDeviceToHost, s));
        VX_CUDA(cudaStreamSynchronize(s));
        e = he;
        if (e > 0) {
            for (DevBuf* b : {&r.tkey, &r.tval, &r.tkey2, &r.tval2}) VX_TRY(b->reserve(size_t(e) * 4, s));
            k_emit_tiles<<<mb, 256, 0, s>>>(order, m, r.bbox.as<int64_t>(), r.off.as<int32_t>(), tiles_x,
                                            r.tkey.as<uint32_t>(), r.tval.as<uint32_t>());
            count_launch();
            int bits = 0;
            while ((1 << bits) < ntl) ++bits;
            bool alt3 = false;
            VX_TRY(radix_sort_pairs(r.tkey.as<uint32_t>(), r.tval.as<uint32_t>(), r.tkey2.as<uint32_t>(),
                                    r.tval2.as<uint32_t>(), e, bits < 1 ? 1 : bits, r.sort_tmp, s, &alt3));
            const uint32_t* tk = alt3 ? r.tkey2.as<uint32_t>() : r.tkey.as<uint32_t>();
            const uint32_t* tv = alt3 ? r.tval2.as<uint32_t>() : r.tval.as<uint32_t>();
            k_tile_ranges<<<unsigned((e + 255) / 256), 256, 0, s>>>(tk, e, r.tstart.as<int32_t>(),
                                                                   r.tend.as<int32_t>());
            count_launch();
            VX_CHECK_LAUNCH();
            RenderArgs ra{r.mean2d.as<double>(), r.cov2d.as<double>(), r.depth.as<double>(),
                          r.bbox.as<int64_t>(), opacity, sh0, order, tv, r.tstart.as<int32_t>(),
                          r.tend.as<int32_t>(), W, H, tiles_x, color, depth, sil};
            k_render_tiles<<<unsigned(ntl), RT2, 0, s>>>(ra);
            count_launch();
            VX_CHECK_LAUNCH();
            return VX_OK;
        }
    }
    // nothing on screen: composited over black, zero depth (renderer.py:190-193)
    VX_CUDA(cudaMemsetAsync(color, 0, size_t(W) * H * 3 * 8, s));
    VX_CUDA(cudaMemsetAsync(depth, 0, size_t(W) * H * 8, s));
    VX_CUDA(cudaMemsetAsync(sil, 0, size_t(W) * H * 8, s));
    return VX_OK;
}

}  // namespace vx
