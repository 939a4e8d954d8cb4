// Gaussian initialisation from solved voxel predictions (splat_init.py:70-148).
//
// One thread per (voxel, subgrid): the n_r^2 points of a subgrid are
// contiguous in the prediction (mesh-grid ordering contract, gpr.py:104-111),
// so a thread streams its block, forms inverse-variance weights
// w = 1/max(var, weight_floor) (splat_init.py:82), the weighted mean (Eq. 6,
// splat_init.py:92-97), the weighted second moment (Eq. 7, 100-114), the
// scale sqrt(clip(diag Phi, 0)) floored, the identity quaternion, and the SH0
// colour of the nearest pixel of the projected mean (117-131, camera.py:65-76)
// falling back to the weighted mean colour (143).
//
// The weight sum uses NumPy's pairwise order and the weighted point / colour
// sums are sequential over rows (ndarray.sum(axis=0) on (k,3)), so positions
// and fallback colours are bit-exact with the reference.
#include <cmath>

#include "vx_common.cuh"
#include "vx_internal.h"

namespace vx {

constexpr double SH0_BASIS = 0.28209479177;   // splat_init.py:22
constexpr int MAX_SUB = 256;                   // n_r^2 with n_s * n_r <= 16

struct SplatArgs {
    const double* pxyz;
    const double* prgb;
    const double* pvar;
    const int32_t* slot_of;    // voxel -> prediction slot (map mode) or null
    const int32_t* voxel_ids;  // (count) voxel ids (map mode) or null
    const int64_t* keys;       // (V,3) map keys (map mode)
    const int64_t* dkeys;      // (count,3) keys (direct mode)
    int64_t count;
    int M, n_s, n_r;
    VxCamera cam;
    const double* image;
    VxSplatConfig cfg;
    VxGaussianOut out;
};

// quaternion (w, x, y, z) of a proper rotation matrix (rows r[0..8])
__device__ void rot_to_quat(const double* R, double* q) {
    const double tr = R[0] + R[4] + R[8];
    if (tr > 0) {
        double s = sqrt(tr + 1.0) * 2.0;
        q[0] = 0.25 * s;
        q[1] = (R[7] - R[5]) / s;
        q[2] = (R[2] - R[6]) / s;
        q[3] = (R[3] - R[1]) / s;
    } else if (R[0] > R[4] && R[0] > R[8]) {
        double s = sqrt(1.0 + R[0] - R[4] - R[8]) * 2.0;
        q[0] = (R[7] - R[5]) / s;
        q[1] = 0.25 * s;
        q[2] = (R[1] + R[3]) / s;
        q[3] = (R[2] + R[6]) / s;
    } else if (R[4] > R[8]) {
        double s = sqrt(1.0 + R[4] - R[0] - R[8]) * 2.0;
        q[0] = (R[2] - R[6]) / s;
        q[1] = (R[1] + R[3]) / s;
        q[2] = 0.25 * s;
        q[3] = (R[5] + R[7]) / s;
    } else {
        double s = sqrt(1.0 + R[8] - R[0] - R[4]) * 2.0;
        q[0] = (R[3] - R[1]) / s;
        q[1] = (R[2] + R[6]) / s;
        q[2] = (R[5] + R[7]) / s;
        q[3] = 0.25 * s;
    }
    double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double sg = q[0] < 0 ? -1.0 : 1.0;
    for (int k = 0; k < 4; ++k) q[k] = sg * q[k] / nrm;
}

// nearest pixel of the projection of p (camera.py:53-76, splat_init.py:124-130);
// leaves rgb (the fallback) untouched when behind the camera or off-image
__device__ void sample_pixel(const VxCamera& cam, const double* image, double px, double py,
                             double pz, double rgb[3]) {
    if (image == nullptr) return;
    const double X = cam.R[0] * px + cam.R[1] * py + cam.R[2] * pz + cam.t[0];
    const double Y = cam.R[3] * px + cam.R[4] * py + cam.R[5] * pz + cam.t[1];
    const double Z = cam.R[6] * px + cam.R[7] * py + cam.R[8] * pz + cam.t[2];
    if (!(Z > 0)) return;
    const double u = xadd(xdiv(xmul(cam.fx, X), Z), cam.cx);
    const double v = xadd(xdiv(xmul(cam.fy, Y), Z), cam.cy);
    if (!(isfinite(u) && isfinite(v))) return;
    const double fu = floor(xadd(u, 0.5)), fv = floor(xadd(v, 0.5));
    if (fu >= 0.0 && fu < double(cam.width) && fv >= 0.0 && fv < double(cam.height)) {
        const int64_t pix = (int64_t(fv) * cam.width + int64_t(fu)) * 3;
        rgb[0] = image[pix];
        rgb[1] = image[pix + 1];
        rgb[2] = image[pix + 2];
    }
}

__global__ void k_init_color(const double* pos, const double* fb, int64_t n, VxCamera cam,
                             const double* image, double* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double rgb[3] = {fb[i * 3], fb[i * 3 + 1], fb[i * 3 + 2]};
    sample_pixel(cam, image, pos[i * 3], pos[i * 3 + 1], pos[i * 3 + 2], rgb);
    for (int d = 0; d < 3; ++d) out[i * 3 + d] = xdiv(xsub(rgb[d], 0.5), SH0_BASIS);
}

int launch_init_color(const double* pos, const double* fallback, int64_t n, const VxCamera& cam,
                      const double* image, double* out, cudaStream_t s) {
    if (n <= 0) return VX_OK;
    k_init_color<<<unsigned((n + 127) / 128), 128, 0, s>>>(pos, fallback, n, cam, image, out);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

template <bool EIGEN, int KT>
__global__ void __launch_bounds__(256) gaussians_kernel(SplatArgs a) {
    // KT = n_r^2 points per subgrid for the common grids (weights in registers);
    // KT = 0: any n_r <= 16 with a runtime loop (weights in local memory)
    constexpr int KW = KT > 0 ? KT : MAX_SUB;
    const int K = KT > 0 ? KT : a.n_r * a.n_r;
    const int nsub = a.n_s * a.n_s;
    const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= a.count * nsub) return;
    const int64_t v = gid / nsub;
    const int b = int(gid - v * nsub);
    int64_t base;
    const int64_t* key;
    if (a.voxel_ids) {
        const int vid = a.voxel_ids[v];
        base = int64_t(a.slot_of[vid]) * a.M;
        key = a.keys + int64_t(vid) * 3;
    } else {
        base = v * a.M;
        key = a.dkeys + v * 3;
    }
    base += int64_t(b) * K;
    const double* P = a.pxyz + base * 3;
    const double* C = a.prgb + base * 3;
    const double* S = a.pvar + base;
    const double wf = a.cfg.weight_floor;
    // w = 1 / max(sigma^2, floor) once per point (splat_init.py:86); np.maximum
    // propagates NaN, variances are finite and clipped here
    double w[KW];
#pragma unroll
    for (int i = 0; i < K; ++i) w[i] = xdiv(1.0, fmax(__ldg(S + i), wf));
    const double wsum = np_pairwise_sum([&](int i) { return w[i]; }, K);
    double px = 0, py = 0, pz = 0, cr = 0, cg = 0, cb = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        px = xadd(px, xmul(__ldg(P + i * 3 + 0), w[i]));
        py = xadd(py, xmul(__ldg(P + i * 3 + 1), w[i]));
        pz = xadd(pz, xmul(__ldg(P + i * 3 + 2), w[i]));
        cr = xadd(cr, xmul(__ldg(C + i * 3 + 0), w[i]));
        cg = xadd(cg, xmul(__ldg(C + i * 3 + 1), w[i]));
        cb = xadd(cb, xmul(__ldg(C + i * 3 + 2), w[i]));
    }
    px = xdiv(px, wsum);
    py = xdiv(py, wsum);
    pz = xdiv(pz, wsum);
    cr = xdiv(cr, wsum);
    cg = xdiv(cg, wsum);
    cb = xdiv(cb, wsum);
    double phi[6] = {0, 0, 0, 0, 0, 0};   // xx xy xz yy yz zz
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const double qx = xsub(__ldg(P + i * 3 + 0), px), qy = xsub(__ldg(P + i * 3 + 1), py),
                     qz = xsub(__ldg(P + i * 3 + 2), pz);
        const double wx = qx * w[i], wy = qy * w[i], wz = qz * w[i];
        phi[0] = fma(wx, qx, phi[0]);
        phi[1] = fma(wx, qy, phi[1]);
        phi[2] = fma(wx, qz, phi[2]);
        phi[3] = fma(wy, qy, phi[3]);
        phi[4] = fma(wy, qz, phi[4]);
        phi[5] = fma(wz, qz, phi[5]);
    }
    for (int j = 0; j < 6; ++j) phi[j] /= wsum;
    const int64_t r = v * nsub + b;
    double scale[3], quat[4] = {1.0, 0.0, 0.0, 0.0};
    if constexpr (EIGEN) {
        // north-star extension: Phi = R diag(s^2) R^T with a right-handed R
        double ev[3], v0[3], V[9];
        eig3_sym(phi, ev, v0, V);
        double det = V[0] * (V[4] * V[8] - V[5] * V[7]) - V[1] * (V[3] * V[8] - V[5] * V[6]) +
                     V[2] * (V[3] * V[7] - V[4] * V[6]);
        if (det < 0) { V[0] = -V[0]; V[3] = -V[3]; V[6] = -V[6]; }
        for (int d = 0; d < 3; ++d) scale[d] = fmax(sqrt(fmax(ev[d], 0.0)), a.cfg.scale_floor);
        rot_to_quat(V, quat);
    } else {
        const double dg[3] = {phi[0], phi[3], phi[5]};
        for (int d = 0; d < 3; ++d) {
            double s = sqrt(dg[d] < 0.0 ? 0.0 : dg[d]);
            scale[d] = s < a.cfg.scale_floor ? a.cfg.scale_floor : s;
        }
    }
    // colour: nearest pixel of the projected mean, else weighted mean colour
    double rgb[3] = {cr, cg, cb};
    sample_pixel(a.cam, a.image, px, py, pz, rgb);
    a.out.position[r * 3 + 0] = px;
    a.out.position[r * 3 + 1] = py;
    a.out.position[r * 3 + 2] = pz;
    for (int d = 0; d < 3; ++d) a.out.scale[r * 3 + d] = scale[d];
    for (int d = 0; d < 4; ++d) a.out.rotation[r * 4 + d] = quat[d];
    a.out.opacity[r] = a.cfg.initial_opacity;
    for (int d = 0; d < 3; ++d) a.out.color[r * 3 + d] = xdiv(xsub(rgb[d], 0.5), SH0_BASIS);
    for (int d = 0; d < 3; ++d) a.out.source_key[r * 3 + d] = key[d];
}

int launch_gaussians(const double* pred_xyz, const double* pred_rgb, const double* pred_var,
                     const int32_t* slot_of, const int32_t* voxel_ids, const int64_t* keys,
                     const int64_t* direct_keys, int64_t count, int M, const VxCamera& cam,
                     const double* image, const VxSplatConfig& cfg, const VxGaussianOut& out,
                     cudaStream_t s) {
    if (count <= 0) return VX_OK;
    if (int64_t(cfg.n_s) * cfg.n_s * cfg.n_r * cfg.n_r != M) {
        set_error("prediction has %d points, expected %d", M, cfg.n_s * cfg.n_s * cfg.n_r * cfg.n_r);
        return VX_E_CONTRACT;
    }
    SplatArgs a{pred_xyz, pred_rgb, pred_var, slot_of, voxel_ids, keys, direct_keys, count,
                M, cfg.n_s, cfg.n_r, cam, image, cfg, out};
    const int64_t threads = count * cfg.n_s * cfg.n_s;
    const unsigned blocks = unsigned((threads + 255) / 256);
    const bool eig = cfg.rotation_mode == VX_ROT_EIGEN;
    switch (cfg.n_r) {
        case 2: eig ? gaussians_kernel<true, 4><<<blocks, 256, 0, s>>>(a)
                    : gaussians_kernel<false, 4><<<blocks, 256, 0, s>>>(a); break;
        case 3: eig ? gaussians_kernel<true, 9><<<blocks, 256, 0, s>>>(a)
                    : gaussians_kernel<false, 9><<<blocks, 256, 0, s>>>(a); break;
        case 4: eig ? gaussians_kernel<true, 16><<<blocks, 256, 0, s>>>(a)
                    : gaussians_kernel<false, 16><<<blocks, 256, 0, s>>>(a); break;
        default: eig ? gaussians_kernel<true, 0><<<blocks, 256, 0, s>>>(a)
                     : gaussians_kernel<false, 0><<<blocks, 256, 0, s>>>(a); break;
    }
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

// ------------------------------------------------------------- PLY vertex records
// formats.py:35-36,126-129: binary little-endian (f32 x, y, z, u8 r, g, b) =
// 15-byte records; positions widen to f64, colours are u8 / 255.0 (exact
// IEEE division, as NumPy's true divide).  Byte loads: records are unaligned.
__global__ void k_decode_ply(const uint8_t* rec, int64_t n, double* xyz, double* rgb) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t* r = rec + i * 15;
    for (int d = 0; d < 3; ++d) {
        const uint32_t b = uint32_t(r[4 * d]) | (uint32_t(r[4 * d + 1]) << 8) |
                           (uint32_t(r[4 * d + 2]) << 16) | (uint32_t(r[4 * d + 3]) << 24);
        xyz[i * 3 + d] = double(__uint_as_float(b));
        rgb[i * 3 + d] = xdiv(double(r[12 + d]), 255.0);
    }
}

int launch_decode_ply(const uint8_t* rec, int64_t n, double* xyz, double* rgb, cudaStream_t s) {
    if (n <= 0) return VX_OK;
    k_decode_ply<<<unsigned((n + 255) / 256), 256, 0, s>>>(rec, n, xyz, rgb);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

// ------------------------------------------------------------- VXSPLAT1 records
// formats.py:25-32: position 3 f8, scale 3 f8, rotation 4 f8, opacity f8,
// color 3 f8, source_key 3 i8 = 136 bytes, little endian, packed.  One thread
// per record assembles it from the SoA fields.
__global__ void k_pack_records(VxGaussianOut in, int64_t count, uint64_t* out) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= count) return;
    uint64_t* o = out + r * 17;
    auto bits = [](double v) { return static_cast<uint64_t>(__double_as_longlong(v)); };
    for (int d = 0; d < 3; ++d) o[d] = bits(in.position[r * 3 + d]);
    for (int d = 0; d < 3; ++d) o[3 + d] = bits(in.scale[r * 3 + d]);
    for (int d = 0; d < 4; ++d) o[6 + d] = bits(in.rotation[r * 4 + d]);
    o[10] = bits(in.opacity[r]);
    for (int d = 0; d < 3; ++d) o[11 + d] = bits(in.color[r * 3 + d]);
    for (int d = 0; d < 3; ++d) o[14 + d] = static_cast<uint64_t>(in.source_key[r * 3 + d]);
}

int launch_pack_records(const VxGaussianOut& in, int64_t count, void* out, cudaStream_t s) {
    if (count <= 0) return VX_OK;
    k_pack_records<<<unsigned((count + 255) / 256), 256, 0, s>>>(in, count,
                                                                 static_cast<uint64_t*>(out));
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

// ------------------------------------------------------------- moments only
__global__ void moments_kernel(const double* pts, const double* w, int64_t G, int k,
                               const double* center, double* pos, double* phi) {
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= G) return;
    const double* P = pts + g * k * 3;
    const double* W = w + g * k;
    const double wsum = np_pairwise_sum([W](int i) { return W[i]; }, k);
    double p[3] = {0, 0, 0};
    for (int i = 0; i < k; ++i)
        for (int d = 0; d < 3; ++d) p[d] = xadd(p[d], xmul(P[i * 3 + d], W[i]));
    for (int d = 0; d < 3; ++d) p[d] = xdiv(p[d], wsum);
    double ctr[3] = {p[0], p[1], p[2]};
    if (center)
        for (int d = 0; d < 3; ++d) ctr[d] = center[g * 3 + d];
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < k; ++i) {
        double q[3];
        for (int d = 0; d < 3; ++d) q[d] = xsub(P[i * 3 + d], ctr[d]);
        for (int r = 0; r < 3; ++r) {
            const double wr = q[r] * W[i];
            for (int c = 0; c < 3; ++c) acc[r * 3 + c] = fma(wr, q[c], acc[r * 3 + c]);
        }
    }
    for (int d = 0; d < 3; ++d) pos[g * 3 + d] = p[d];
    for (int e = 0; e < 9; ++e) phi[g * 9 + e] = acc[e] / wsum;
}

int launch_moments(const double* pts, const double* w, int64_t G, int k, const double* center,
                   double* pos, double* phi, cudaStream_t s) {
    if (G <= 0) return VX_OK;
    moments_kernel<<<unsigned((G + 127) / 128), 128, 0, s>>>(pts, w, G, k, center, pos, phi);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

}  // namespace vx
