// Batched per-voxel Gaussian-process regression, FP64, sm_100a.
//
// Replaces gpr.py:57-311 (select_value_axis, make_mesh_grid, kernel_matrix,
// gpr_solve, densify_frame's per-voxel body) and voxel_map.py:242-261 /
// 344-355 (apply_prediction's fold-back and reclassification).
//
// Stages, chosen per training-set size n (size buckets):
//
//  * PCA prepass (thread per voxel): centroid, 3x3 covariance, Jacobi eigen,
//    value axis + degeneracy test (gpr.py:57-78) and the pairwise mean of the
//    targets (gpr.py:291).  Decouples the serial per-voxel work from the
//    solve kernels and lets degenerate voxels drop out before bucketing.
//  * warp kernel (n <= 16 / 32 / 64): ONE WARP per voxel, no CTA barriers.
//    The warp builds A = K + diag(noise) column-major in its shared-memory
//    slice, factorises it left-looking (lanes = rows, dot products against
//    the broadcast pivot row, one __syncwarp per column), then every lane
//    owns one right-hand side column of [f | K*] per pass (ceil((m+1)/32)
//    passes) and runs a right-looking forward substitution with the column
//    in registers and L columns read as 16-byte pairs:
//        w = L^-1 k*_c,  sigma^2_c = 1 - |w|^2,  mu_c = w . (L^-1 f).
//    K* is never materialised: for the SE kernel on the voxel's regular grid
//    k*(x_i, g) = exp(-lam dx^2) exp(-lam dy^2) is separable, so the warp
//    tabulates 2 * n * (n_s n_r) exponentials instead of n * (n_s n_r)^2.
//  * generic kernel (any n): one CTA per voxel, A/L (column-major) and W in a
//    per-CTA global workspace (L2-resident), left-looking Cholesky and a
//    row-blocked forward substitution.  Serves the Livox-style tail and
//    re-fits whose raw ∪ pseudo training sets grow past 64 points.
//
// Both write the prediction (points, colours, clipped variances) into the
// voxel's prediction slot — which is also the pseudo-observation set of its
// next solve — and update the lifecycle state in the same kernel.
#include <atomic>
#include <cfloat>
#include <cstdlib>
#include <cmath>

#include "vx_common.cuh"
#include "vx_internal.h"

namespace vx {

// Diagnostics build (-DVX_PHASE_TIMING): thread 0 of every tile-kernel CTA
// adds the SM clock cycles of each phase of each voxel to g_phase_cycles,
// read back (and reset) by the extra export vx_phase_cycles
// (tools/phase_timing.py).  Compiled out otherwise.
#ifdef VX_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[20];
#define VX_PHASE(id, t0)                                                                  \
    do {                                                                                  \
        if (threadIdx.x == 0) {                                                           \
            const long long t1_ = clock64();                                              \
            atomicAdd(&g_phase_cycles[id], (unsigned long long)(t1_ - (t0)));             \
            (t0) = t1_;                                                                   \
        }                                                                                 \
    } while (0)
#else
#define VX_PHASE(id, t0) do { } while (0)
#endif

constexpr int MAX_MM = 16;   // n_s * n_r <= 16 (grid 4..16 per axis sweep)

// ---------------------------------------------------------------------------
// problem-mode arguments (gpr_solve_batch)
// ---------------------------------------------------------------------------
struct ProblemArgs {
    const int32_t* items;
    int32_t num_items;
    const int64_t* x_off;
    const int64_t* q_off;
    const double* x;
    const double* f;
    const double* noise;
    const double* xs;
    const double* lam;
    double jitter;
    int kernel;
    double* mu;
    double* var;
    double* full;
    const int64_t* full_off;
    uint8_t* status;
};

// ---------------------------------------------------------------------------
// PCA prepass: one thread per candidate voxel
// ---------------------------------------------------------------------------
__device__ __forceinline__ const double* train_point(const VoxelSolveArgs& a, int r, int cnt,
                                                     int64_t off, int slot) {
    return r < cnt ? a.raw_xyz + (off + r) * 3
                   : a.pred_xyz + (int64_t(slot) * a.M + (r - cnt)) * 3;
}

__global__ void __launch_bounds__(128) k_pca_prepass(VoxelSolveArgs a, int S, long long* buckets) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const int vid = a.cand_voxel[s];
    const int n = a.cand_n[s];
    const int cnt = a.raw_count[vid];
    const int64_t off = a.raw_offset[vid];
    const int slot = a.pred_slot[vid];
    const int ax = pca_value_axis([&](int r) { return train_point(a, r, cnt, off, slot); }, n);
    a.cand_axis[s] = int8_t(ax);
    if (ax < 0) {
        a.cand_status[s] = VX_ST_DEGENERATE;
        const uint8_t st = a.state[vid];
        a.cand_before[s] = st;
        a.cand_after[s] = st;
        return;
    }
    const double sum = np_pairwise_sum(
        [&](int i) { return train_point(a, i, cnt, off, slot)[ax]; }, n);
    a.cand_meanf[s] = xdiv(sum, double(n));                    // f.mean() (gpr.py:291)
    agg_add(reinterpret_cast<unsigned long long*>(buckets), bucket_of(n));
}

__global__ void k_bucket_items(const int32_t* cand_n, const int8_t* cand_axis, int S, int32_t* items,
                               const long long* base, long long* fill) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S || cand_axis[s] < 0) return;
    const int b = bucket_of(cand_n[s]);
    const long long pos = agg_add(reinterpret_cast<unsigned long long*>(fill), b);
    items[base[b] + pos] = int32_t(s);
}

// ---------------------------------------------------------------------------
// warp-per-voxel kernel (n <= NMAX, NMAX in {16, 32, 64})
// ---------------------------------------------------------------------------
// per-warp shared-memory slice (doubles), LD = NMAX (even: 16-byte columns)
struct WarpLayout {
    int X, F, NZ, L, INV, EA, EB, MU, VAR, COL, BI, GC, total;
    __host__ __device__ WarpLayout(int NMAX, int mm, int m, bool voxel) {
        int o = 0;
        X = o; o += 2 * NMAX;
        F = o; o += NMAX;
        NZ = o; o += NMAX;            // noise, later z = L^-1 f
        L = o; o += NMAX * NMAX;
        INV = o; o += NMAX;
        EA = o; EB = o;
        MU = VAR = COL = BI = GC = o;
        if (voxel) {
            EA = o; o += NMAX * mm;
            EB = o; o += NMAX * mm;
            MU = o; o += m;
            VAR = o; o += m;
            COL = o; o += 3 * m;
            BI = o; o += (m + 1) / 2;  // int32 pairs
            GC = o; o += 2 * mm;       // grid coordinates c0[mm], c1[mm]
        }
        total = (o + 1) & ~1;
    }
};

// triangular index -> (i, j), j <= i
__device__ __forceinline__ void tri_decode(int idx, int* i, int* j) {
    int r = int((sqrt(8.0 * idx + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= idx) ++r;
    while (r * (r + 1) / 2 > idx) --r;
    *i = r;
    *j = idx - r * (r + 1) / 2;
}

template <int NMAX, bool VOXEL>
__global__ void __launch_bounds__(128, NMAX <= 16 ? 5 : (NMAX <= 24 ? 4 : (NMAX <= 32 ? 3 : 1))) gpr_warp_kernel(VoxelSolveArgs va, ProblemArgs pa, int mmax,
                                                       int mm) {
    extern __shared__ __align__(16) double smem[];
    constexpr int LD = NMAX;
    constexpr int RPL = NMAX > 32 ? 2 : 1;          // Cholesky rows per lane
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const WarpLayout lay(NMAX, mm, mmax, VOXEL);
    double* base = smem + size_t(wib) * lay.total;
    double* X = base + lay.X;
    double* F = base + lay.F;
    double* NZ = base + lay.NZ;
    double* L = base + lay.L;
    double* INV = base + lay.INV;
    const int num_items = VOXEL ? va.num_items : pa.num_items;

    for (int it = blockIdx.x * wpb + wib; it < num_items; it += gridDim.x * wpb) {
        int n, m, s, vid = 0, cnt = 0, slot = 0, axis = 2;
        int64_t off = 0, xo = 0, qo = 0;
        double lam, jitter, mean_f = 0.0;
        int kind;
        double lo0 = 0, lo1 = 0, sp0 = 0, sp1 = 0;
        if constexpr (VOXEL) {
            s = va.items[it];
            vid = va.cand_voxel[s];
            n = va.cand_n[s];
            cnt = va.raw_count[vid];
            off = va.raw_offset[vid];
            slot = va.pred_slot[vid];
            m = va.M;
            lam = va.lam;
            jitter = va.jitter;
            kind = va.kernel;
            axis = va.cand_axis[s];
            mean_f = va.cand_meanf[s];
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            // ---- stage raw ∪ pseudo (voxel_map.py:196-200), split by axis
            for (int r = lane; r < n; r += 32) {
                const double* p = train_point(va, r, cnt, off, slot);
                X[2 * r] = p[pa_];
                X[2 * r + 1] = p[pb_];
                F[r] = xsub(p[axis], mean_f);
                NZ[r] = r < cnt ? va.sensor_var : va.pred_var[int64_t(slot) * m + (r - cnt)];
            }
            // ---- voxel grid (gpr.py:104-120, 262-266): lo + ((i + 0.5) * (hi - lo)) / m
            lo0 = xmul(double(va.keys[int64_t(vid) * 3 + pa_]), va.voxel_size);
            lo1 = xmul(double(va.keys[int64_t(vid) * 3 + pb_]), va.voxel_size);
            sp0 = xsub(xadd(lo0, va.voxel_size), lo0);
            sp1 = xsub(xadd(lo1, va.voxel_size), lo1);
            // grid coordinates c_r = lo + ((r + 0.5) * (hi - lo)) / m, once per voxel
            if (lane < 2 * mm) {
                const int which = lane >= mm, r = lane - which * mm;
                base[lay.GC + lane] = xadd(which ? lo1 : lo0,
                                           xdiv(xmul(double(r) + 0.5, which ? sp1 : sp0), double(mm)));
            }
            __syncwarp();
            const double* GC = base + lay.GC;
            if (kind == VX_KERNEL_SE) {
                double* EA = base + lay.EA;
                double* EB = base + lay.EB;
                // lane = (table, training row); rows >= n get zeros (padding)
                for (int e = lane; e < 2 * NMAX; e += 32) {
                    const int which = e / NMAX, i = e - which * NMAX;
                    double* T = (which ? EB : EA) + i * mm;
                    if (i < n) {
                        const double xi = X[2 * i + which];
                        for (int r = 0; r < mm; ++r) {
                            const double g = GC[which * mm + r];
                            const double d = xsub(xi, g);
                            T[r] = exp(xmul(-lam, xmul(d, d)));
                        }
                    } else {
                        for (int r = 0; r < mm; ++r) T[r] = 0.0;
                    }
                }
            }
        } else {
            s = pa.items[it];
            xo = pa.x_off[s];
            qo = pa.q_off[s];
            n = int(pa.x_off[s + 1] - xo);
            m = int(pa.q_off[s + 1] - qo);
            lam = pa.lam[s];
            jitter = pa.jitter;
            kind = pa.kernel;
            for (int r = lane; r < n; r += 32) {
                X[2 * r] = pa.x[(xo + r) * 2];
                X[2 * r + 1] = pa.x[(xo + r) * 2 + 1];
                F[r] = pa.f[xo + r];
                NZ[r] = pa.noise[xo + r];
            }
        }
        __syncwarp();

        // ---- A = K + diag(noise), Cholesky, one jitter retry (gpr.py:184-194)
        bool ok = false;
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            const double jit = attempt ? jitter : 0.0;
            // whole NMAX x NMAX column-major square: the live lower triangle, zeros
            // elsewhere, so the forward substitution can run unguarded on
            // padding rows (their right-hand sides and 1/L_ii are zero)
            for (int e = lane; e < NMAX * NMAX; e += 32) {
                const int j = e / NMAX, i = e - j * NMAX;
                double v = 0.0;
                if (i < n && j <= i) {
                    if (i == j) {
                        v = xadd(1.0, NZ[i]);          // K_ii = exp(-lam*0) = 1, + noise
                        if (jit != 0.0) v = xadd(v, jit);
                    } else {
                        v = kernel_value(kind, lam,
                                         dist2_exact(X[2 * i], X[2 * i + 1], X[2 * j], X[2 * j + 1]));
                    }
                }
                L[e] = v;
            }
            if (lane < NMAX) INV[lane] = 0.0;
            if (NMAX > 32 && lane + 32 < NMAX) INV[lane + 32] = 0.0;
            __syncwarp();
            ok = true;
            for (int j = 0; j < n; ++j) {
                double sv[RPL];
#pragma unroll
                for (int rr = 0; rr < RPL; ++rr) {
                    const int i = j + lane + 32 * rr;
                    double s0 = 0.0, s1 = 0.0;
                    if (i < n) {
                        s0 = L[j * LD + i];
                        int k = 0;
                        for (; k + 1 < j; k += 2) {
                            s0 = fma(-L[k * LD + i], L[k * LD + j], s0);
                            s1 = fma(-L[(k + 1) * LD + i], L[(k + 1) * LD + j], s1);
                        }
                        if (k < j) s0 = fma(-L[k * LD + i], L[k * LD + j], s0);
                    }
                    sv[rr] = s0 + s1;
                }
                const double d = __shfl_sync(FULL, sv[0], 0);   // pivot row j is lane 0
                if (!(d > 0.0)) {                                 // dpotrf: pivot <= 0 or NaN
                    ok = false;
                    break;
                }
                const double inv = rsqrt(d);                      // dpotf2 scales by 1/ajj
                const double ljj = d * inv;
#pragma unroll
                for (int rr = 0; rr < RPL; ++rr) {
                    const int i = j + lane + 32 * rr;
                    if (i < n) L[j * LD + i] = (i == j) ? ljj : sv[rr] * inv;
                }
                if (lane == 0) INV[j] = inv;
                __syncwarp();
            }
            __syncwarp();
        }
        if (!ok) {
            if (lane == 0) {
                if constexpr (VOXEL) {
                    va.cand_status[s] = VX_ST_CHOL_FAIL;
                    const uint8_t st = va.state[vid];
                    va.cand_before[s] = st;
                    va.cand_after[s] = st;
                } else {
                    pa.status[s] = VX_ST_CHOL_FAIL;
                }
            }
            __syncwarp();
            continue;
        }

        // ---- forward substitution, lane = one column of [f | K*] per pass
        const int ncols = m + 1;
        const int passes = (ncols + 31) >> 5;
        const double* EA = base + lay.EA;
        const double* EB = base + lay.EB;
        for (int pass = 0; pass < passes; ++pass) {
            const int c = pass * 32 + lane;
            const bool active = c < ncols;
            const int q = c - 1;
            double g0 = 0, g1 = 0;
            int ri = 0, si = 0;
            if (active && c > 0) {
                if constexpr (VOXEL) {
                    const int nr = va.n_r, ns = va.n_s, nr2 = nr * nr;
                    const int sr = q / (ns * nr2);
                    const int rem = q - sr * ns * nr2;
                    const int sc = rem / nr2;
                    const int rem2 = rem - sc * nr2;
                    const int fr = rem2 / nr, fc = rem2 - fr * nr;
                    ri = sr * nr + fr;
                    si = sc * nr + fc;
                    g0 = base[lay.GC + ri];
                    g1 = base[lay.GC + mm + si];
                } else {
                    g0 = pa.xs[(qo + q) * 2];
                    g1 = pa.xs[(qo + q) * 2 + 1];
                }
            }
            double b[NMAX];
            if (VOXEL && kind == VX_KERNEL_SE && c > 0) {
                // separable tables are zero on padding rows
#pragma unroll
                for (int i = 0; i < NMAX; ++i) b[i] = active ? EA[i * mm + ri] * EB[i * mm + si] : 0.0;
            } else {
#pragma unroll
                for (int i = 0; i < NMAX; ++i) {
                    double r = 0.0;
                    if (i < n && active) {
                        if (c == 0) r = F[i];
                        else r = kernel_value(kind, lam, dist2_exact(X[2 * i], X[2 * i + 1], g0, g1));
                    }
                    b[i] = r;
                }
            }
            double ss = 0.0;
#pragma unroll
            for (int i = 0; i < NMAX; ++i) {
                if (i < n) {                                   // uniform: skips dead columns
                    const double w = b[i] * INV[i];
                    ss = fma(w, w, ss);
                    const double* Lc = L + i * LD;            // column i: L(r, i) at Lc[r]
#pragma unroll
                    for (int r = (i + 1) & ~1; r < NMAX; r += 2) {   // zero rows >= n
                        const double2 l2 = *reinterpret_cast<const double2*>(Lc + r);
                        b[r] = fma(-l2.x, w, b[r]);
                        b[r + 1] = fma(-l2.y, w, b[r + 1]);
                    }
                    b[i] = w;                                  // (r == i above touched a dead value)
                }
            }
            if (pass == 0) {
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < NMAX; ++i) NZ[i] = b[i];   // z = L^-1 f (0 on padding)
                }
                __syncwarp();
            }
            if (active && c > 0) {
                double mu0 = 0.0, mu1 = 0.0;
#pragma unroll
                for (int i = 0; i < NMAX; i += 2) {
                    mu0 = fma(b[i], NZ[i], mu0);
                    mu1 = fma(b[i + 1], NZ[i + 1], mu1);
                }
                const double mu = mu0 + mu1;
                const double var = 1.0 - ss;
                if constexpr (VOXEL) {
                    base[lay.MU + q] = xadd(mu, mean_f);
                    base[lay.VAR + q] = var < 0.0 ? 0.0 : var;      // np.clip(., 0, None)
                    // nearest training point in the parameter plane (gpr.py:304-305)
                    double best = INFINITY;
                    int bi = 0;
                    for (int i = 0; i < n; ++i) {
                        const double d2 = dist2_exact(g0, g1, X[2 * i], X[2 * i + 1]);
                        if (d2 < best) { best = d2; bi = i; }
                    }
                    reinterpret_cast<int*>(base + lay.BI)[q] = bi;
                } else {
                    pa.mu[qo + q] = mu;
                    pa.var[qo + q] = var;
                }
            }
        }
        if constexpr (VOXEL) {
            __syncwarp();
            double* COL = base + lay.COL;
            const int* BI = reinterpret_cast<const int*>(base + lay.BI);
            // read phase: colours may come from the previous prediction of this voxel
            for (int q = lane; q < m; q += 32) {
                const int bi = BI[q];
                const double* cs = bi < cnt ? va.raw_rgb + (off + bi) * 3
                                            : va.pred_rgb + (int64_t(slot) * m + (bi - cnt)) * 3;
                COL[q * 3] = cs[0];
                COL[q * 3 + 1] = cs[1];
                COL[q * 3 + 2] = cs[2];
            }
            __syncwarp();
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            double* oxyz = va.pred_xyz + int64_t(slot) * m * 3;
            double* orgb = va.pred_rgb + int64_t(slot) * m * 3;
            double* ovar = va.pred_var + int64_t(slot) * m;
            const int nr = va.n_r, ns = va.n_s, nr2 = nr * nr;
            for (int q = lane; q < m; q += 32) {
                const int sr = q / (ns * nr2);
                const int rem = q - sr * ns * nr2;
                const int sc = rem / nr2;
                const int rem2 = rem - sc * nr2;
                const int fr = rem2 / nr, fc = rem2 - fr * nr;
                double pos[3];
                pos[axis] = base[lay.MU + q];
                pos[pa_] = base[lay.GC + sr * nr + fr];
                pos[pb_] = base[lay.GC + mm + sc * nr + fc];
                oxyz[q * 3] = pos[0];
                oxyz[q * 3 + 1] = pos[1];
                oxyz[q * 3 + 2] = pos[2];
                orgb[q * 3] = COL[q * 3];
                orgb[q * 3 + 1] = COL[q * 3 + 1];
                orgb[q * 3 + 2] = COL[q * 3 + 2];
                ovar[q] = base[lay.VAR + q];
            }
            if (lane == 0) {
                const double* V = base + lay.VAR;
                const double mv = xdiv(np_pairwise_sum([V](int i) { return V[i]; }, m), double(m));
                const uint8_t before = va.state[vid];
                const uint8_t after = mv <= va.eta ? VX_CONVERGED : VX_ACTIVE;
                va.state[vid] = after;
                va.value_axis[vid] = int8_t(axis);
                va.has_pred[vid] = 1;
                va.cand_status[s] = VX_ST_OK;
                va.cand_before[s] = before;
                va.cand_after[s] = after;
            }
        } else {
            if (lane == 0) pa.status[s] = VX_ST_OK;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// generic kernel: any n, one CTA (GB threads) per problem, global workspace
// ---------------------------------------------------------------------------
constexpr int GB = 128;

struct GenericWork {
    double* base;
    int64_t per_cta;   // doubles
    int nmax, mmax;
};

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = (l < GB / 32) ? red[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(FULL, r, o);
        if (l == 0) red[0] = r;
    }
    __syncthreads();
    r = red[0];
    __syncthreads();
    return r;
}

template <bool VOXEL>
__global__ void __launch_bounds__(GB) gpr_generic_kernel(VoxelSolveArgs va, ProblemArgs pa,
                                                         GenericWork gw) {
    const int tid = threadIdx.x;
    double* ws = gw.base + int64_t(blockIdx.x) * gw.per_cta;
    const int NM = gw.nmax, MM = gw.mmax;
    double* P3 = ws;                     // max(NM,MM)*3: points, later colour stash
    double* X = P3 + int64_t(NM > MM ? NM : MM) * 3;    // NM*2
    double* F = X + int64_t(NM) * 2;     // NM
    double* NZ = F + NM;                 // NM
    double* VAR = NZ + NM;               // MM
    double* L = VAR + MM;                // NM*NM column-major (ld = n)
    double* W = L + int64_t(NM) * NM;    // NM*(MM+1) row-major (ld = m+1)

    const int num_items = VOXEL ? va.num_items : pa.num_items;
    for (int it = blockIdx.x; it < num_items; it += gridDim.x) {
        int n, m, s = 0, vid = 0, cnt = 0, slot = 0, axis = 2, mm = 1;
        int64_t off = 0, xo = 0, qo = 0;
        double lam, jitter, mean_f = 0.0;
        int kind;
        if constexpr (VOXEL) {
            s = va.items[it];
            vid = va.cand_voxel[s];
            n = va.cand_n[s];
            cnt = va.raw_count[vid];
            off = va.raw_offset[vid];
            slot = va.pred_slot[vid];
            m = va.M;
            mm = va.n_s * va.n_r;
            lam = va.lam;
            jitter = va.jitter;
            kind = va.kernel;
            axis = va.cand_axis[s];
            mean_f = va.cand_meanf[s];
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            for (int r = tid; r < n; r += GB) {
                const double* p = train_point(va, r, cnt, off, slot);
                X[2 * r] = p[pa_];
                X[2 * r + 1] = p[pb_];
                F[r] = xsub(p[axis], mean_f);
                NZ[r] = r < cnt ? va.sensor_var : va.pred_var[int64_t(slot) * m + (r - cnt)];
            }
        } else {
            s = pa.items[it];
            xo = pa.x_off[s];
            qo = pa.q_off[s];
            n = int(pa.x_off[s + 1] - xo);
            m = int(pa.q_off[s + 1] - qo);
            lam = pa.lam[s];
            jitter = pa.jitter;
            kind = pa.kernel;
            for (int r = tid; r < n; r += GB) {
                X[2 * r] = pa.x[(xo + r) * 2];
                X[2 * r + 1] = pa.x[(xo + r) * 2 + 1];
                F[r] = pa.f[xo + r];
                NZ[r] = pa.noise[xo + r];
            }
        }
        __syncthreads();

        // ---- Cholesky, column-major L (L(i,j) at L[j*n+i]), one jitter retry
        bool ok = false;
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            const double jit = attempt ? jitter : 0.0;
            for (int j = 0; j < n; ++j) {
                for (int i = j + tid; i < n; i += GB) {
                    double v;
                    if (i == j) {
                        v = xadd(1.0, NZ[i]);
                        if (jit != 0.0) v = xadd(v, jit);
                    } else {
                        v = kernel_value(kind, lam,
                                         dist2_exact(X[2 * i], X[2 * i + 1], X[2 * j], X[2 * j + 1]));
                    }
                    L[int64_t(j) * n + i] = v;
                }
            }
            __syncthreads();
            ok = true;
            for (int j = 0; j < n; ++j) {
                for (int i = j + tid; i < n; i += GB) {
                    double s0 = L[int64_t(j) * n + i], s1 = 0.0;
                    int k = 0;
                    for (; k + 1 < j; k += 2) {
                        s0 = fma(-L[int64_t(k) * n + i], L[int64_t(k) * n + j], s0);
                        s1 = fma(-L[int64_t(k + 1) * n + i], L[int64_t(k + 1) * n + j], s1);
                    }
                    if (k < j) s0 = fma(-L[int64_t(k) * n + i], L[int64_t(k) * n + j], s0);
                    L[int64_t(j) * n + i] = s0 + s1;
                }
                __syncthreads();
                const double d = L[int64_t(j) * n + j];
                if (!(d > 0.0)) { ok = false; break; }
                const double ljj = sqrt(d);
                for (int i = j + 1 + tid; i < n; i += GB) L[int64_t(j) * n + i] /= ljj;
                __syncthreads();
                if (tid == 0) L[int64_t(j) * n + j] = ljj;
                __syncthreads();
            }
            __syncthreads();
        }
        if (!ok) {
            if (tid == 0) {
                if constexpr (VOXEL) {
                    va.cand_status[s] = VX_ST_CHOL_FAIL;
                    uint8_t st = va.state[vid];
                    va.cand_before[s] = st;
                    va.cand_after[s] = st;
                } else {
                    pa.status[s] = VX_ST_CHOL_FAIL;
                }
            }
            __syncthreads();
            continue;
        }

        // ---- forward substitution, rows blocked by 8, W row-major (ld = m+1)
        double lo0 = 0, lo1 = 0, sp0 = 0, sp1 = 0;
        if constexpr (VOXEL) {
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            lo0 = xmul(double(va.keys[vid * 3 + pa_]), va.voxel_size);
            lo1 = xmul(double(va.keys[vid * 3 + pb_]), va.voxel_size);
            sp0 = xsub(xadd(lo0, va.voxel_size), lo0);
            sp1 = xsub(xadd(lo1, va.voxel_size), lo1);
        }
        const int ldw = m + 1;
        for (int c = tid; c < ldw; c += GB) {
            double g0 = 0, g1 = 0;
            if (c > 0) {
                const int q = c - 1;
                if constexpr (VOXEL) {
                    const int nr2 = va.n_r * va.n_r;
                    const int sr = q / (va.n_s * nr2);
                    const int rem = q - sr * va.n_s * nr2;
                    const int sc = rem / nr2;
                    const int rem2 = rem - sc * nr2;
                    const int fr = rem2 / va.n_r, fc = rem2 - fr * va.n_r;
                    g0 = xadd(lo0, xdiv(xmul(double(sr * va.n_r + fr) + 0.5, sp0), double(mm)));
                    g1 = xadd(lo1, xdiv(xmul(double(sc * va.n_r + fc) + 0.5, sp1), double(mm)));
                } else {
                    g0 = pa.xs[(qo + q) * 2];
                    g1 = pa.xs[(qo + q) * 2 + 1];
                }
            }
            for (int i0 = 0; i0 < n; i0 += 8) {
                const int rb = min(8, n - i0);
                double acc[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    if (r < rb) {
                        const int i = i0 + r;
                        acc[r] = (c == 0) ? F[i]
                                          : kernel_value(kind, lam,
                                                         dist2_exact(X[2 * i], X[2 * i + 1], g0, g1));
                    } else {
                        acc[r] = 0.0;
                    }
                }
                for (int j = 0; j < i0; ++j) {
                    const double wj = W[int64_t(j) * ldw + c];
                    const double* Lj = L + int64_t(j) * n + i0;
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (r < rb) acc[r] = fma(-Lj[r], wj, acc[r]);
                }
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    if (r < rb) {
                        const int i = i0 + r;
                        double b = acc[r];
#pragma unroll
                        for (int r2 = 0; r2 < r; ++r2) b = fma(-L[int64_t(i0 + r2) * n + i], acc[r2], b);
                        acc[r] = b / L[int64_t(i) * n + i];
                        W[int64_t(i) * ldw + c] = acc[r];
                    }
                }
            }
        }
        __syncthreads();
        for (int c = 1 + tid; c < ldw; c += GB) {
            const int q = c - 1;
            double ss = 0.0, mu0 = 0.0, mu1 = 0.0;
            for (int i = 0; i < n; ++i) {
                const double wi = W[int64_t(i) * ldw + c];
                ss = fma(wi, wi, ss);
                if (i & 1) mu1 = fma(wi, W[int64_t(i) * ldw], mu1);
                else mu0 = fma(wi, W[int64_t(i) * ldw], mu0);
            }
            const double mu = mu0 + mu1, var = 1.0 - ss;
            if constexpr (VOXEL) {
                VAR[q] = var < 0.0 ? 0.0 : var;
                W[c] = mu;   // stash mu in row 0 of its own column (only its owner reads it)
            } else {
                pa.mu[qo + q] = mu;
                pa.var[qo + q] = var;
            }
        }
        __syncthreads();
        if constexpr (!VOXEL) {
            if (pa.full != nullptr) {
                // Sigma* = Kss - W^T W (gpr.py:202-204)
                double* out = pa.full + pa.full_off[s];
                for (int e = tid; e < m * m; e += GB) {
                    const int a = e / m, b = e - a * m;
                    double kab = kernel_value(kind, lam,
                                              dist2_exact(pa.xs[(qo + a) * 2], pa.xs[(qo + a) * 2 + 1],
                                                          pa.xs[(qo + b) * 2], pa.xs[(qo + b) * 2 + 1]));
                    double acc0 = 0.0;
                    for (int i = 0; i < n; ++i)
                        acc0 = fma(W[int64_t(i) * ldw + 1 + a], W[int64_t(i) * ldw + 1 + b], acc0);
                    out[e] = kab - acc0;
                }
            }
            if (tid == 0) pa.status[s] = VX_ST_OK;
            __syncthreads();
            continue;
        } else {
            // ---- epilogue (gpr.py:303-310): points, nearest colour, clip
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            // read phase: the previous prediction may be a colour source
            for (int q = tid; q < m; q += GB) {
                const int nr2 = va.n_r * va.n_r;
                const int sr = q / (va.n_s * nr2);
                const int rem = q - sr * va.n_s * nr2;
                const int sc = rem / nr2;
                const int rem2 = rem - sc * nr2;
                const int fr = rem2 / va.n_r, fc = rem2 - fr * va.n_r;
                const double g0 = xadd(lo0, xdiv(xmul(double(sr * va.n_r + fr) + 0.5, sp0), double(mm)));
                const double g1 = xadd(lo1, xdiv(xmul(double(sc * va.n_r + fc) + 0.5, sp1), double(mm)));
                double best = INFINITY;
                int bi = 0;
                for (int i = 0; i < n; ++i) {
                    double d2 = dist2_exact(g0, g1, X[2 * i], X[2 * i + 1]);
                    if (d2 < best) { best = d2; bi = i; }
                }
                const double* cs = bi < cnt ? va.raw_rgb + (off + bi) * 3
                                            : va.pred_rgb + (int64_t(slot) * m + (bi - cnt)) * 3;
                // stash point (P3 rows are free now) and colour (X no longer needed after
                // everyone has finished the argmin -> use P3 for both)
                P3[q * 3 + 0] = cs[0];
                P3[q * 3 + 1] = cs[1];
                P3[q * 3 + 2] = cs[2];
            }
            __syncthreads();
            for (int q = tid; q < m; q += GB) {
                const int nr2 = va.n_r * va.n_r;
                const int sr = q / (va.n_s * nr2);
                const int rem = q - sr * va.n_s * nr2;
                const int sc = rem / nr2;
                const int rem2 = rem - sc * nr2;
                const int fr = rem2 / va.n_r, fc = rem2 - fr * va.n_r;
                const double g0 = xadd(lo0, xdiv(xmul(double(sr * va.n_r + fr) + 0.5, sp0), double(mm)));
                const double g1 = xadd(lo1, xdiv(xmul(double(sc * va.n_r + fc) + 0.5, sp1), double(mm)));
                double pos[3];
                pos[axis] = xadd(W[q + 1], mean_f);
                pos[pa_] = g0;
                pos[pb_] = g1;
                const int64_t pr = int64_t(slot) * m + q;
                va.pred_xyz[pr * 3 + 0] = pos[0];
                va.pred_xyz[pr * 3 + 1] = pos[1];
                va.pred_xyz[pr * 3 + 2] = pos[2];
                va.pred_rgb[pr * 3 + 0] = P3[q * 3 + 0];
                va.pred_rgb[pr * 3 + 1] = P3[q * 3 + 1];
                va.pred_rgb[pr * 3 + 2] = P3[q * 3 + 2];
                va.pred_var[pr] = VAR[q];
            }
            __syncthreads();
            if (tid == 0) {
                double mv = xdiv(np_pairwise_sum([VAR](int i) { return VAR[i]; }, m), double(m));
                uint8_t before = va.state[vid];
                uint8_t after = mv <= va.eta ? VX_CONVERGED : VX_ACTIVE;
                va.state[vid] = after;
                va.value_axis[vid] = int8_t(axis);
                va.has_pred[vid] = 1;
                va.cand_status[s] = VX_ST_OK;
                va.cand_before[s] = before;
                va.cand_after[s] = after;
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// blocked CTA kernel (n > 64): one voxel per CTA of CT threads
// ---------------------------------------------------------------------------
// Buffers live in one workspace that is the CTA's dynamic shared memory when
// it fits, else a per-CTA slice of global memory (L2-resident):
//   Lp   packed column-major lower triangle; column j starts at row (j & ~1)
//        and is padded to an even length so L(r, j) pairs with even r are
//        16-byte aligned (element (i, j) at off[j] + i - (j & ~1))
//   W    row-major n x WLD right-hand-side block of the current column pass
// Cholesky: left-looking by panels of P = 8 columns.  Each thread owns rows
//   and updates P accumulators per previous column k with one load of L(i,k)
//   and four 16-byte loads of L(J,k) (8 FMAs : 5 loads); the P x P diagonal
//   block is then factorised redundantly in every thread's registers (same
//   values -> same pivot decision, no extra barrier) and applied to the
//   thread's rows.  dpotrf's failure rule, one jitter retry.
// Forward substitution: a thread owns one column of [f | K*]; rows go in
//   chunks of CH = 16 held in registers; each previous row j contributes
//   acc(R) -= L(R, j) w_j with 8 paired 16-byte loads per 16 FMAs.
constexpr int CT = 96;
constexpr int PNL = 8;
constexpr int CH = 16;

struct CtaLayout {
    int64_t X, F, NZ, INV, EA, EB, MU, VAR, COL, BI, OFF, Lp, W, total;
    int n_pad, wld;
    __host__ __device__ CtaLayout(int n, int mm, int m, bool voxel) {
        n_pad = (n + 1) & ~1;
        const int cols = m + 1;
        wld = cols < CT ? cols : CT;
        int64_t o = 0;
        X = o; o += 2 * n_pad;
        F = o; o += n_pad;
        NZ = o; o += n_pad;            // noise, later z = L^-1 f
        INV = o; o += n_pad;
        EA = EB = MU = VAR = COL = BI = o;
        if (voxel) {
            EA = o; o += int64_t(n_pad) * mm;
            EB = o; o += int64_t(n_pad) * mm;
            MU = o; o += m + (m & 1);
            VAR = o; o += m + (m & 1);
            COL = o; o += 3 * m + (m & 1);
            BI = o; o += (m + 1) / 2 + ((m + 1) / 2 & 1);
        }
        OFF = o; o += (n_pad + 2) / 2 + 2;    // int32 column offsets (as doubles)
        o = (o + 1) & ~int64_t(1);
        Lp = o;
        const int64_t hp = n_pad / 2;
        o += 2 * (hp * n_pad - hp * (hp - 1)) + 2 * PNL + 4;
        o = (o + 1) & ~int64_t(1);
        W = o; o += int64_t(n_pad + CH) * wld;
        total = (o + 1) & ~int64_t(1);
    }
};

template <bool VOXEL>
__global__ void __launch_bounds__(CT) gpr_cta_kernel(VoxelSolveArgs va, ProblemArgs pa, int nmax,
                                                     int mmax, int mm, double* gwork, int64_t per_cta) {
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x;
    const CtaLayout lay(nmax, mm, mmax, VOXEL);
    double* base = gwork ? gwork + int64_t(blockIdx.x) * per_cta : smem;
    double* X = base + lay.X;
    double* F = base + lay.F;
    double* NZ = base + lay.NZ;
    double* INV = base + lay.INV;
    int* OFF = reinterpret_cast<int*>(base + lay.OFF);
    double* Lp = base + lay.Lp;
    double* W = base + lay.W;
    const int num_items = VOXEL ? va.num_items : pa.num_items;

    for (int it = blockIdx.x; it < num_items; it += gridDim.x) {
        int n, m, s, vid = 0, cnt = 0, slot = 0, axis = 2;
        int64_t off = 0, xo = 0, qo = 0;
        double lam, jitter, mean_f = 0.0;
        int kind;
        double lo0 = 0, lo1 = 0, sp0 = 0, sp1 = 0;
        if constexpr (VOXEL) {
            s = va.items[it];
            vid = va.cand_voxel[s];
            n = va.cand_n[s];
            cnt = va.raw_count[vid];
            off = va.raw_offset[vid];
            slot = va.pred_slot[vid];
            m = va.M;
            lam = va.lam;
            jitter = va.jitter;
            kind = va.kernel;
            axis = va.cand_axis[s];
            mean_f = va.cand_meanf[s];
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            for (int r = tid; r < n; r += CT) {
                const double* p = train_point(va, r, cnt, off, slot);
                X[2 * r] = p[pa_];
                X[2 * r + 1] = p[pb_];
                F[r] = xsub(p[axis], mean_f);
                NZ[r] = r < cnt ? va.sensor_var : va.pred_var[int64_t(slot) * m + (r - cnt)];
            }
            lo0 = xmul(double(va.keys[int64_t(vid) * 3 + pa_]), va.voxel_size);
            lo1 = xmul(double(va.keys[int64_t(vid) * 3 + pb_]), va.voxel_size);
            sp0 = xsub(xadd(lo0, va.voxel_size), lo0);
            sp1 = xsub(xadd(lo1, va.voxel_size), lo1);
            __syncthreads();
            if (kind == VX_KERNEL_SE) {
                double* EA = base + lay.EA;
                double* EB = base + lay.EB;
                for (int e = tid; e < 2 * n * mm; e += CT) {
                    const int which = e >= n * mm;
                    const int rem = e - which * n * mm;
                    const int i = rem / mm, r = rem - i * mm;
                    const double lo = which ? lo1 : lo0, sp = which ? sp1 : sp0;
                    const double g = xadd(lo, xdiv(xmul(double(r) + 0.5, sp), double(mm)));
                    const double d = xsub(X[2 * i + which], g);
                    (which ? EB : EA)[i * mm + r] = exp(xmul(-lam, xmul(d, d)));
                }
            }
        } else {
            s = pa.items[it];
            xo = pa.x_off[s];
            qo = pa.q_off[s];
            n = int(pa.x_off[s + 1] - xo);
            m = int(pa.q_off[s + 1] - qo);
            lam = pa.lam[s];
            jitter = pa.jitter;
            kind = pa.kernel;
            for (int r = tid; r < n; r += CT) {
                X[2 * r] = pa.x[(xo + r) * 2];
                X[2 * r + 1] = pa.x[(xo + r) * 2 + 1];
                F[r] = pa.f[xo + r];
                NZ[r] = pa.noise[xo + r];
            }
        }
        const int n_pad = (n + 1) & ~1;
        // packed column offsets: columns 2u and 2u+1 both hold n_pad - 2u rows
        for (int j = tid; j <= n; j += CT) {
            const int u = j >> 1;
            int o = 2 * (u * n_pad - u * (u - 1));
            if (j & 1) o += n_pad - 2 * u;
            OFF[j] = o;
        }
        __syncthreads();
        auto Lat = [&](int i, int j) -> double& { return Lp[OFF[j] + i - (j & ~1)]; };

        // ---- A = K + diag(noise), panel Cholesky, one jitter retry
        bool ok = false;
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            const double jit = attempt ? jitter : 0.0;
            for (int j = 0; j < n; ++j) {
                for (int i = j + tid; i < n; i += CT) {
                    double v;
                    if (i == j) {
                        v = xadd(1.0, NZ[i]);
                        if (jit != 0.0) v = xadd(v, jit);
                    } else {
                        v = kernel_value(kind, lam,
                                         dist2_exact(X[2 * i], X[2 * i + 1], X[2 * j], X[2 * j + 1]));
                    }
                    Lat(i, j) = v;
                }
            }
            __syncthreads();
            ok = true;
            for (int j0 = 0; j0 < n; j0 += PNL) {
                const int pw = min(PNL, n - j0);
                // phase 1: A(i, J) -= sum_{k<j0} L(i,k) L(J,k) for the thread's rows
                for (int i = j0 + tid; i < n; i += CT) {
                    double acc[PNL];
#pragma unroll
                    for (int q = 0; q < PNL; ++q) acc[q] = (q < pw && j0 + q <= i) ? Lat(i, j0 + q) : 0.0;
                    for (int k = 0; k < j0; ++k) {
                        const double* col = Lp + OFF[k] - (k & ~1);
                        const double lik = col[i];
                        const double2* lj = reinterpret_cast<const double2*>(col + j0);
#pragma unroll
                        for (int q = 0; q < PNL; q += 2) {
                            const double2 v = lj[q >> 1];
                            acc[q] = fma(-lik, v.x, acc[q]);
                            acc[q + 1] = fma(-lik, v.y, acc[q + 1]);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < PNL; ++q)
                        if (q < pw && j0 + q <= i) Lat(i, j0 + q) = acc[q];
                }
                __syncthreads();
                // phase 2: factor the diagonal block redundantly, then the thread's rows
                double d[PNL][PNL];
#pragma unroll
                for (int a = 0; a < PNL; ++a)
#pragma unroll
                    for (int b = 0; b < PNL; ++b)
                        d[a][b] = (a < pw && b <= a) ? Lat(j0 + a, j0 + b) : 0.0;
                double inv[PNL];
#pragma unroll
                for (int c = 0; c < PNL; ++c) {
                    if (c < pw && ok) {
                        double sdiag = d[c][c];
#pragma unroll
                        for (int k = 0; k < c; ++k) sdiag = fma(-d[c][k], d[c][k], sdiag);
                        if (!(sdiag > 0.0)) {
                            ok = false;
                        } else {
                            const double lcc = sqrt(sdiag);
                            inv[c] = 1.0 / lcc;
                            d[c][c] = lcc;
#pragma unroll
                            for (int r = c + 1; r < PNL; ++r) {
                                double v = d[r][c];
#pragma unroll
                                for (int k = 0; k < c; ++k) v = fma(-d[r][k], d[c][k], v);
                                d[r][c] = v * inv[c];
                            }
                        }
                    }
                }
                if (!ok) break;                          // uniform: same values in every thread
                // rows below the block: L(i, J) = A(i, J) L_JJ^-T
                for (int i = j0 + pw + tid; i < n; i += CT) {
                    double v[PNL];
#pragma unroll
                    for (int c = 0; c < PNL; ++c) {
                        if (c < pw) {
                            double t = Lat(i, j0 + c);
#pragma unroll
                            for (int k = 0; k < c; ++k) t = fma(-v[k], d[c][k], t);
                            v[c] = t * inv[c];
                        }
                    }
#pragma unroll
                    for (int c = 0; c < PNL; ++c)
                        if (c < pw) Lat(i, j0 + c) = v[c];
                }
#pragma unroll
                for (int a = 0; a < PNL; ++a) {          // static indices keep d[][] in registers
                    if (a == tid && a < pw) {
#pragma unroll
                        for (int b = 0; b <= a; ++b) Lat(j0 + a, j0 + b) = d[a][b];
                        INV[j0 + a] = inv[a];
                    }
                }
                __syncthreads();
            }
            __syncthreads();
        }
        if (!ok) {
            if (tid == 0) {
                if constexpr (VOXEL) {
                    va.cand_status[s] = VX_ST_CHOL_FAIL;
                    const uint8_t st = va.state[vid];
                    va.cand_before[s] = st;
                    va.cand_after[s] = st;
                } else {
                    pa.status[s] = VX_ST_CHOL_FAIL;
                }
            }
            __syncthreads();
            continue;
        }

        // ---- forward substitution in row chunks, one column per thread
        const int ncols = m + 1;
        const int wld = lay.wld;
        const double* EA = base + lay.EA;
        const double* EB = base + lay.EB;
        for (int c0 = 0; c0 < ncols; c0 += wld) {
            const int c = c0 + tid;
            const bool active = tid < wld && c < ncols;
            const int q = c - 1;
            double g0 = 0, g1 = 0;
            int ri = 0, si = 0;
            if (active && c > 0) {
                if constexpr (VOXEL) {
                    const int nr = va.n_r, ns = va.n_s, nr2 = nr * nr;
                    const int sr = q / (ns * nr2);
                    const int rem = q - sr * ns * nr2;
                    const int sc = rem / nr2;
                    const int rem2 = rem - sc * nr2;
                    const int fr = rem2 / nr, fc = rem2 - fr * nr;
                    ri = sr * nr + fr;
                    si = sc * nr + fc;
                    g0 = xadd(lo0, xdiv(xmul(double(ri) + 0.5, sp0), double(mm)));
                    g1 = xadd(lo1, xdiv(xmul(double(si) + 0.5, sp1), double(mm)));
                } else {
                    g0 = pa.xs[(qo + q) * 2];
                    g1 = pa.xs[(qo + q) * 2 + 1];
                }
            }
            double ss = 0.0;
            if (active) {
                for (int k0 = 0; k0 < n; k0 += CH) {
                    double acc[CH];
#pragma unroll
                    for (int r = 0; r < CH; ++r) {
                        const int i = k0 + r;
                        double v = 0.0;
                        if (i < n) {
                            if (c == 0) v = F[i];
                            else if (VOXEL && kind == VX_KERNEL_SE) v = EA[i * mm + ri] * EB[i * mm + si];
                            else v = kernel_value(kind, lam, dist2_exact(X[2 * i], X[2 * i + 1], g0, g1));
                        }
                        acc[r] = v;
                    }
                    for (int j = 0; j < k0; ++j) {
                        const double wj = W[int64_t(j) * wld + tid];
                        const double2* lc =
                            reinterpret_cast<const double2*>(Lp + OFF[j] - (j & ~1) + k0);
#pragma unroll
                        for (int r = 0; r < CH; r += 2) {
                            const double2 l2 = lc[r >> 1];
                            acc[r] = fma(-l2.x, wj, acc[r]);
                            acc[r + 1] = fma(-l2.y, wj, acc[r + 1]);
                        }
                    }
#pragma unroll
                    for (int r = 0; r < CH; ++r) {
                        const int i = k0 + r;
                        if (i < n) {
                            const double w = acc[r] * INV[i];
                            const double* lc = Lp + OFF[i] - (i & ~1) + k0;   // column i, rows k0..
#pragma unroll
                            for (int r2 = (r + 1) & ~1; r2 < CH; r2 += 2) {
                                const double2 l2 = *reinterpret_cast<const double2*>(lc + r2);
                                acc[r2] = fma(-l2.x, w, acc[r2]);
                                acc[r2 + 1] = fma(-l2.y, w, acc[r2 + 1]);
                            }
                            acc[r] = w;
                            ss = fma(w, w, ss);
                            W[int64_t(i) * wld + tid] = w;
                        }
                    }
                }
            }
            __syncthreads();
            if (c0 == 0 && tid == 0) {
                for (int i = 0; i < n; ++i) NZ[i] = W[int64_t(i) * wld];   // z = L^-1 f
            }
            __syncthreads();
            if (active && c > 0) {
                double mu0 = 0.0, mu1 = 0.0;
                int i = 0;
                for (; i + 1 < n; i += 2) {
                    mu0 = fma(W[int64_t(i) * wld + tid], NZ[i], mu0);
                    mu1 = fma(W[int64_t(i + 1) * wld + tid], NZ[i + 1], mu1);
                }
                if (i < n) mu0 = fma(W[int64_t(i) * wld + tid], NZ[i], mu0);
                const double mu = mu0 + mu1;
                const double var = 1.0 - ss;
                if constexpr (VOXEL) {
                    base[lay.MU + q] = xadd(mu, mean_f);
                    base[lay.VAR + q] = var < 0.0 ? 0.0 : var;
                    double best = INFINITY;
                    int bi = 0;
                    for (int t = 0; t < n; ++t) {
                        const double d2 = dist2_exact(g0, g1, X[2 * t], X[2 * t + 1]);
                        if (d2 < best) { best = d2; bi = t; }
                    }
                    reinterpret_cast<int*>(base + lay.BI)[q] = bi;
                } else {
                    pa.mu[qo + q] = mu;
                    pa.var[qo + q] = var;
                }
            }
            __syncthreads();
        }
        if constexpr (VOXEL) {
            double* COL = base + lay.COL;
            const int* BI = reinterpret_cast<const int*>(base + lay.BI);
            for (int q = tid; q < m; q += CT) {
                const int bi = BI[q];
                const double* cs = bi < cnt ? va.raw_rgb + (off + bi) * 3
                                            : va.pred_rgb + (int64_t(slot) * m + (bi - cnt)) * 3;
                COL[q * 3] = cs[0];
                COL[q * 3 + 1] = cs[1];
                COL[q * 3 + 2] = cs[2];
            }
            __syncthreads();
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            double* oxyz = va.pred_xyz + int64_t(slot) * m * 3;
            double* orgb = va.pred_rgb + int64_t(slot) * m * 3;
            double* ovar = va.pred_var + int64_t(slot) * m;
            const int nr = va.n_r, ns = va.n_s, nr2 = nr * nr;
            for (int q = tid; q < m; q += CT) {
                const int sr = q / (ns * nr2);
                const int rem = q - sr * ns * nr2;
                const int sc = rem / nr2;
                const int rem2 = rem - sc * nr2;
                const int fr = rem2 / nr, fc = rem2 - fr * nr;
                double pos[3];
                pos[axis] = base[lay.MU + q];
                pos[pa_] = xadd(lo0, xdiv(xmul(double(sr * nr + fr) + 0.5, sp0), double(mm)));
                pos[pb_] = xadd(lo1, xdiv(xmul(double(sc * nr + fc) + 0.5, sp1), double(mm)));
                oxyz[q * 3] = pos[0];
                oxyz[q * 3 + 1] = pos[1];
                oxyz[q * 3 + 2] = pos[2];
                orgb[q * 3] = COL[q * 3];
                orgb[q * 3 + 1] = COL[q * 3 + 1];
                orgb[q * 3 + 2] = COL[q * 3 + 2];
                ovar[q] = base[lay.VAR + q];
            }
            if (tid == 0) {
                const double* V = base + lay.VAR;
                const double mv = xdiv(np_pairwise_sum([V](int i) { return V[i]; }, m), double(m));
                const uint8_t before = va.state[vid];
                const uint8_t after = mv <= va.eta ? VX_CONVERGED : VX_ACTIVE;
                va.state[vid] = after;
                va.value_axis[vid] = int8_t(axis);
                va.has_pred[vid] = 1;
                va.cand_status[s] = VX_ST_OK;
                va.cand_before[s] = before;
                va.cand_after[s] = after;
            }
        } else {
            if (tid == 0) pa.status[s] = VX_ST_OK;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// DMMA tile kernel (33 <= n <= 128): FP64 tensor cores (mma.m8n8k4.f64)
// ---------------------------------------------------------------------------
// One voxel per CTA of NW warps.  The training set is padded to n8 = 8*ceil(n/8)
// rows with an identity block (padding rows have zero right-hand sides, so they
// do not change any result).  A lives column-major in shared memory (LD = n8+4
// keeps DMMA fragment loads at two wavefronts).
//  Cholesky: left-looking by 8-column panels.  The panel update
//    A(i >= j0, J) -= L(i, <j0) L(J, <j0)^T is a GEMM done with DMMA 8x8x4
//    (row tiles spread over the warps); warp 0 factors the 8x8 diagonal block
//    with shuffles (dpotrf failure rule); the rows below are solved against it.
//  Forward substitution: right-looking with the whole right-hand-side block
//    resident in registers as DMMA accumulators: warp w owns CTW column tiles
//    (8 columns each) of [f | K*]; for each row block k it solves the 8x8
//    diagonal system with shuffles, converts W_k to B fragments and updates all
//    later row blocks with DMMA.  No shared-memory W, no CTA barrier inside.
__device__ __forceinline__ void dmma_acc(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// warp-per-voxel DMMA kernel (voxel mode, n <= NMAX, NMAX in {16, 24, 32})
// ---------------------------------------------------------------------------
// One warp per voxel, no CTA barriers inside the voxel loop.
//   * A = K + diag(noise): the strict lower triangle is filled compactly
//     (lane = entry, from a per-CTA (i, j) table), then lane i holds row i of
//     A in registers and the warp factorises right-looking: column j is
//     scaled in registers, published to shared memory (column-major L) and
//     read back as 16-byte broadcasts for the rank-1 update of the rows.
//   * lane c forms column c of L^-1 by substitution; L^-1 is stored row-major
//     over L's slot and its fragments stay in registers for the whole voxel.
//   * W^T = [f | K*]^T L^-T with m8n8k4 DMMA, 8 right-hand sides per tile:
//     the A operand K*(i, q) = EA[ri(q)][i] * EB[si(q)][i] comes from the
//     separable tables (stored transposed so a lane's four rows are
//     immediate offsets), the B operand is the L^-1 fragment.  Accumulator
//     rows are queries, so sigma^2_q = 1 - |w_q|^2 and mu_q = w_q . z
//     (z = L^-1 f, row 0 of tile 0) reduce over the 4 lanes of a row.
// 11 independent column tiles per voxel at n* = 81.
template <int NMAX>
#ifndef W16_MINB
#define W16_MINB 6
#define W24_MINB 4
#define W32_MINB 3
#endif
__global__ void __launch_bounds__(128, NMAX <= 16 ? W16_MINB : (NMAX <= 24 ? W24_MINB : W32_MINB))
gpr_wdmma_kernel(VoxelSolveArgs va, int mmax, int mm) {
    extern __shared__ __align__(16) double smem[];
    constexpr int LD = NMAX;
    constexpr int NRB = NMAX / 8;         // 8-row blocks
    constexpr int NKS = NMAX / 4;         // k-chunks of 4
    constexpr int NA = NRB * (NRB + 1);   // fragments of the lower-triangular L^-1
    constexpr int NTRI = NMAX * (NMAX - 1) / 2;
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int wib = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    const WarpLayout lay(NMAX, mm, mmax, true);
    const int ncols = va.M + 1;
    const int ntiles = (ncols + 7) >> 3;
    // per-CTA tables: ONE/ZERO rows, column c of [f | K*] -> (ri, si) of
    // query c - 1, strict-lower-triangle entry e -> (i, j)
    double* ONE = smem + size_t(wpb) * lay.total;
    double* ZERO = ONE + NMAX;
    int* QRI = reinterpret_cast<int*>(ZERO + NMAX);
    int* QSI = QRI + 8 * ntiles;
    int* TRI = QSI + 8 * ntiles;
    for (int c = threadIdx.x; c < 8 * ntiles; c += blockDim.x) {
        int ri = -1, si = -1;
        if (c >= 1 && c < ncols) {
            const int q = c - 1;
            const int nr = va.n_r, ns = va.n_s, nr2 = nr * nr;
            const int sr = q / (ns * nr2);
            const int rem = q - sr * ns * nr2;
            const int sc = rem / nr2;
            const int rem2 = rem - sc * nr2;
            const int fr = rem2 / nr, fc = rem2 - fr * nr;
            ri = sr * nr + fr;
            si = sc * nr + fc;
        }
        QRI[c] = ri;
        QSI[c] = si;
    }
    for (int e = threadIdx.x; e < NTRI; e += blockDim.x) {
        int r, j;
        tri_decode(e, &r, &j);                 // e = r (r + 1) / 2 + j, j <= r
        TRI[e] = (r + 1) | (j << 8);           // row i = r + 1 > j
    }
    for (int i = threadIdx.x; i < NMAX; i += blockDim.x) {
        ONE[i] = 1.0;
        ZERO[i] = 0.0;
    }
    __syncthreads();
    double* base = smem + size_t(wib) * lay.total;
    double* X = base + lay.X;
    double* F = base + lay.F;
    double* NZ = base + lay.NZ;
    double* L = base + lay.L;
    double* INV = base + lay.INV;
    double* EA = base + lay.EA;           // EA[r * NMAX + i] = exp(-lam (x_i - c_r)^2)
    double* EB = base + lay.EB;
    double* GC = base + lay.GC;
    double* MU = base + lay.MU;
    double* VAR = base + lay.VAR;

    for (int it = blockIdx.x * wpb + wib; it < va.num_items; it += gridDim.x * wpb) {
        const int s = va.items[it];
        const int vid = va.cand_voxel[s];
        const int n = va.cand_n[s];
        const int cnt = va.raw_count[vid];
        const int64_t off = va.raw_offset[vid];
        const int slot = va.pred_slot[vid];
        const int m = va.M;
        const double lam = va.lam;
        const int kind = va.kernel;
        const int axis = va.cand_axis[s];
        const double mean_f = va.cand_meanf[s];
        const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
        // ---- stage raw ∪ pseudo (voxel_map.py:196-200), split by axis; pad with zeros
        for (int r = lane; r < NMAX; r += 32) {
            if (r < n) {
                const double* p = train_point(va, r, cnt, off, slot);
                X[2 * r] = p[pa_];
                X[2 * r + 1] = p[pb_];
                F[r] = xsub(p[axis], mean_f);
                NZ[r] = r < cnt ? va.sensor_var : va.pred_var[int64_t(slot) * m + (r - cnt)];
            } else {
                X[2 * r] = X[2 * r + 1] = F[r] = NZ[r] = 0.0;
            }
        }
        // ---- voxel grid (gpr.py:104-120, 262-266): lo + ((i + 0.5) * (hi - lo)) / m
        const double lo0 = xmul(double(va.keys[int64_t(vid) * 3 + pa_]), va.voxel_size);
        const double lo1 = xmul(double(va.keys[int64_t(vid) * 3 + pb_]), va.voxel_size);
        const double sp0 = xsub(xadd(lo0, va.voxel_size), lo0);
        const double sp1 = xsub(xadd(lo1, va.voxel_size), lo1);
        if (lane < 2 * mm) {
            const int which = lane >= mm, r = lane - which * mm;
            GC[lane] = xadd(which ? lo1 : lo0, xdiv(xmul(double(r) + 0.5, which ? sp1 : sp0), double(mm)));
        }
        __syncwarp();
        // ---- separable tables (SE), transposed: lane = (table, training row)
        if (kind == VX_KERNEL_SE) {
            for (int e = lane; e < 2 * NMAX; e += 32) {
                const int which = e / NMAX, i = e - which * NMAX;
                double* T = (which ? EB : EA) + i;
                if (i < n) {
                    const double xi = X[2 * i + which];
                    for (int r = 0; r < mm; ++r) {
                        const double d = xsub(xi, GC[which * mm + r]);
                        T[r * NMAX] = exp(xmul(-lam, xmul(d, d)));
                    }
                } else {
                    for (int r = 0; r < mm; ++r) T[r * NMAX] = 0.0;
                }
            }
        }

        // ---- A = K + diag(noise), right-looking Cholesky in registers, one
        //      jitter retry (gpr.py:184-194)
        bool ok = false;
        double a[NMAX];
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            const double jit = attempt ? va.jitter : 0.0;
            const int ntri = n * (n - 1) / 2;
            for (int e = lane; e < ntri; e += 32) {
                const int ij = TRI[e];
                const int i = ij & 0xff, j = ij >> 8;
                L[j * LD + i] = kernel_value(kind, lam, dist2_exact(X[2 * i], X[2 * i + 1], X[2 * j], X[2 * j + 1]));
            }
            double dg = 1.0;                      // padding rows: identity
            if (lane < n) {
                dg = xadd(1.0, NZ[lane]);         // K_ii = exp(-lam*0) = 1, + noise
                if (jit != 0.0) dg = xadd(dg, jit);
            }
            __syncwarp();
            // NMAX == 16: lanes 16 + c carry the augmented row e_c^T through the
            // same right-looking sweep, which leaves column c of L^-1 in their
            // registers (the forward substitution L x = e_c in the order and
            // roundings of the separate lane-per-column pass it replaces)
#pragma unroll
            for (int k = 0; k < NMAX; ++k) {
                double v = 0.0;
                if (NMAX == 16 && lane >= 16) v = (k == lane - 16) ? 1.0 : 0.0;
                else if (k == lane) v = dg;
                else if (k < lane && lane < n) v = L[k * LD + lane];
                a[k] = v;
            }
            __syncwarp();
            ok = true;
#pragma unroll
            for (int j = 0; j < NMAX; ++j) {
                if (j >= n) break;
                const double piv = __shfl_sync(FULL, a[j], j);
                if (!(piv > 0.0)) {               // dpotrf: pivot <= 0 or NaN
                    ok = false;
                    break;
                }
                const double inv = rsqrt(piv);    // dpotf2 scales by 1/ajj
                const double l = (lane == j) ? piv * inv : a[j] * inv;
                a[j] = l;
                if (lane < NMAX) L[j * LD + lane] = l;   // rows < j: unused upper entries
                if (lane == 0) INV[j] = inv;
                __syncwarp();
                if (j + 1 < NMAX) {
                    const double* Lj = L + j * LD;
                    int k = j + 1;
                    if (k & 1) {
                        a[k] = fma(-l, Lj[k], a[k]);
                        ++k;
                    }
#pragma unroll
                    for (; k + 1 < NMAX; k += 2) {
                        const double2 lk = *reinterpret_cast<const double2*>(Lj + k);
                        a[k] = fma(-l, lk.x, a[k]);
                        a[k + 1] = fma(-l, lk.y, a[k + 1]);
                    }
                }
            }
            __syncwarp();
        }
        if (!ok) {
            if (lane == 0) {
                va.cand_status[s] = VX_ST_CHOL_FAIL;
                const uint8_t st = va.state[vid];
                va.cand_before[s] = st;
                va.cand_after[s] = st;
            }
            __syncwarp();
            continue;
        }

        // ---- L^-1, lane c = column c (rows >= n and columns >= n stay zero);
        //      NMAX == 16: already in lanes 16..31 (padding columns c >= n
        //      hold e_c, which meets only zero rows of [f | K*])
        if constexpr (NMAX == 16) {
            if (lane >= 16) {
#pragma unroll
                for (int r = 0; r < NMAX; ++r) L[r * LD + (lane - 16)] = a[r];
            }
            __syncwarp();
        } else {
            double x[NMAX];
#pragma unroll
            for (int r = 0; r < NMAX; ++r) {
                double v = 0.0;
                if (r < n) {
                    double acc = (r == lane) ? 1.0 : 0.0;
#pragma unroll
                    for (int k = 0; k < r; ++k) acc = fma(-L[k * LD + r], x[k], acc);
                    v = (r < lane) ? 0.0 : acc * INV[r];
                }
                x[r] = v;
            }
            __syncwarp();
            if (lane < NMAX) {
#pragma unroll
                for (int r = 0; r < NMAX; ++r) L[r * LD + lane] = x[r];   // row-major L^-1
            }
            __syncwarp();
        }
        double bf[NA];                 // B = L^-T fragments: block (cb, s), s <= 2 cb + 1
        {
            int t = 0;
#pragma unroll
            for (int cb = 0; cb < NRB; ++cb)
#pragma unroll
                for (int s2 = 0; s2 < 2 * cb + 2; ++s2) bf[t++] = L[(8 * cb + g) * LD + 4 * s2 + tig];
        }

        // ---- W^T = [f | K*]^T L^-T by tiles of 8 right-hand sides
        double zr[NRB][2];
        for (int ct = 0; ct < ntiles; ++ct) {
            const int col = 8 * ct + g;              // accumulator row = right-hand side
            const int ri = QRI[col], si = QSI[col];
            double af[NKS];
            if (kind == VX_KERNEL_SE) {
                const double* pA = ri >= 0 ? EA + ri * NMAX : (col == 0 ? F : ZERO);
                const double* pB = si >= 0 ? EB + si * NMAX : ONE;
#pragma unroll
                for (int s2 = 0; s2 < NKS; ++s2) af[s2] = pA[4 * s2 + tig] * pB[4 * s2 + tig];
            } else {
#pragma unroll
                for (int s2 = 0; s2 < NKS; ++s2) {
                    const int row = 4 * s2 + tig;
                    double v = 0.0;
                    if (ri >= 0) {
                        if (row < n) v = kernel_value(kind, lam, dist2_exact(X[2 * row], X[2 * row + 1],
                                                                             GC[ri], GC[mm + si]));
                    } else if (col == 0) {
                        v = F[row];
                    }
                    af[s2] = v;
                }
            }
            double c[NRB][2];
            {
                int t = 0;
#pragma unroll
                for (int cb = 0; cb < NRB; ++cb) {
                    c[cb][0] = c[cb][1] = 0.0;
#pragma unroll
                    for (int s2 = 0; s2 < 2 * cb + 2; ++s2) dmma_acc(c[cb][0], c[cb][1], af[s2], bf[t++]);
                }
            }
            if (ct == 0) {
                // row 0 of tile 0 is z^T = (L^-1 f)^T: lanes 0..3 hold z(8 cb + 2 tig + e)
#pragma unroll
                for (int cb = 0; cb < NRB; ++cb) {
                    zr[cb][0] = __shfl_sync(FULL, c[cb][0], tig);
                    zr[cb][1] = __shfl_sync(FULL, c[cb][1], tig);
                }
            }
            double ss = 0.0, mu = 0.0;
#pragma unroll
            for (int cb = 0; cb < NRB; ++cb) {
                ss = fma(c[cb][0], c[cb][0], ss);
                ss = fma(c[cb][1], c[cb][1], ss);
                mu = fma(c[cb][0], zr[cb][0], mu);
                mu = fma(c[cb][1], zr[cb][1], mu);
            }
            ss += __shfl_xor_sync(FULL, ss, 1);
            mu += __shfl_xor_sync(FULL, mu, 1);
            ss += __shfl_xor_sync(FULL, ss, 2);
            mu += __shfl_xor_sync(FULL, mu, 2);
            if (tig == 0 && col >= 1 && col < ncols) {
                const double var = 1.0 - ss;
                MU[col - 1] = xadd(mu, mean_f);
                VAR[col - 1] = var < 0.0 ? 0.0 : var;      // np.clip(., 0, None)
            }
        }

        // ---- nearest training point in the parameter plane (gpr.py:304-305), colours
        int* BI = reinterpret_cast<int*>(base + lay.BI);
        // three queries per lane in one pass over the training points (each
        // point's coordinates loaded once, three independent min chains)
        for (int q0 = lane; q0 < m; q0 += 96) {
            double g0[3], g1[3], best[3];
            int bi[3];
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int q = q0 + 32 * u < m ? q0 + 32 * u : q0;
                g0[u] = GC[QRI[q + 1]];
                g1[u] = GC[mm + QSI[q + 1]];
                best[u] = INFINITY;
                bi[u] = 0;
            }
            for (int i = 0; i < n; ++i) {
                const double2 xi = *reinterpret_cast<const double2*>(X + 2 * i);
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const double d2 = dist2_exact(g0[u], g1[u], xi.x, xi.y);
                    if (d2 < best[u]) { best[u] = d2; bi[u] = i; }
                }
            }
#pragma unroll
            for (int u = 0; u < 3; ++u)
                if (q0 + 32 * u < m) BI[q0 + 32 * u] = bi[u];
        }
        __syncwarp();
        double* COL = base + lay.COL;
        // read phase: colours may come from the previous prediction of this voxel
        for (int q = lane; q < m; q += 32) {
            const int bi = BI[q];
            const double* cs = bi < cnt ? va.raw_rgb + (off + bi) * 3
                                        : va.pred_rgb + (int64_t(slot) * m + (bi - cnt)) * 3;
            COL[q * 3] = cs[0];
            COL[q * 3 + 1] = cs[1];
            COL[q * 3 + 2] = cs[2];
        }
        __syncwarp();
        double* oxyz = va.pred_xyz + int64_t(slot) * m * 3;
        double* orgb = va.pred_rgb + int64_t(slot) * m * 3;
        double* ovar = va.pred_var + int64_t(slot) * m;
        for (int q = lane; q < m; q += 32) {
            // assemble_points (gpr.py:89-97) with selects (no local-memory array)
            const double pv = MU[q], p0 = GC[QRI[q + 1]], p1 = GC[mm + QSI[q + 1]];
            oxyz[q * 3] = axis == 0 ? pv : (pa_ == 0 ? p0 : p1);
            oxyz[q * 3 + 1] = axis == 1 ? pv : (pa_ == 1 ? p0 : p1);
            oxyz[q * 3 + 2] = axis == 2 ? pv : (pa_ == 2 ? p0 : p1);
            orgb[q * 3] = COL[q * 3];
            orgb[q * 3 + 1] = COL[q * 3 + 1];
            orgb[q * 3 + 2] = COL[q * 3 + 2];
            ovar[q] = VAR[q];
        }
        const double mv = xdiv(warp_pairwise_sum(VAR, m), double(m));
        if (lane == 0) {
            const uint8_t before = va.state[vid];
            const uint8_t after = mv <= va.eta ? VX_CONVERGED : VX_ACTIVE;
            va.state[vid] = after;
            va.value_axis[vid] = int8_t(axis);
            va.has_pred[vid] = 1;
            va.cand_status[s] = VX_ST_OK;
            va.cand_before[s] = before;
            va.cand_after[s] = after;
        }
        __syncwarp();
    }
}

// Packed block-column storage of the lower triangle: block column kb (columns
// 8kb..8kb+7) holds rows 8kb..n8-1 column-major with leading dimension
// ldb = rows + 4 (rows a multiple of 8, so ldb = 4 or 12 mod 16 doubles): the
// four columns of a DMMA fragment load land on disjoint banks per half-warp.
__host__ __device__ inline int tile_ldb(int n8, int kb) {
    return n8 - 8 * kb + 4;
}
__host__ __device__ inline int tile_packed(int n8) {
    int t = 0;
    for (int kb = 0; kb < n8 / 8; ++kb) t += 8 * tile_ldb(n8, kb);
    return t;
}

struct TileLayout {
    int L, CO, LINV, LDG, X, F, NZ, INV, Z, EA, EB, MU, VAR, COL, FLAG, GC, QT, W, total;
    __host__ __device__ TileLayout(int N8, int mm, int mcols, int mmax, bool voxel,
                                   bool with_w = false) {
        int o = 0;
        L = o; o += tile_packed(N8);
        CO = o; o += N8 / 2 + 1;        // int32 column offsets: L(i, j) = L[CO[j] + i]
        LDG = o; o += N8 * 8;           // factored 8x8 diagonal blocks, row-major
        LINV = LDG;                     // then their inverses, in place
        X = o; o += 2 * N8;
        F = o; o += N8;
        NZ = o; o += N8;
        INV = o; o += N8;
        Z = o; o += N8;
        EA = EB = COL = o;
        if (voxel) {
            EA = o; o += N8 * mm;
            EB = o; o += N8 * mm;
            COL = o; o += 3 * mmax + 1;
        }
        MU = o; o += mcols;
        VAR = o; o += mcols;
        FLAG = o; o += 2;
        GC = o; o += 2 * MAX_MM;        // grid coordinates of both parameter axes
        QT = o; o += mcols;             // int32 (ri, si) of column c = q + 1
        o = (o + 1) & ~1;
        W = o;
        if (with_w) o += N8 * mcols;    // row-major right-hand-side block (big kernel)
        total = (o + 1) & ~1;
    }
};

// A = K + diag(noise) (+ jitter on the retry), identity-padded to n8 rows,
// into the packed lower triangle (gpr.py:184-186).  Thread = lower-triangle
// entry (single-precision root + fix-up decode); two entries per iteration
// with branch-free selects so their exp chains interleave.
__device__ __forceinline__ void team_fill_matrix(double* L, const int* CO, const double* X,
                                                 const double* NZ, int n, int n8, int kind,
                                                 double lam, double jit, int tid, int nt) {
    const int tot = n8 * (n8 + 1) / 2;
    for (int e0 = tid; e0 < tot; e0 += 2 * nt) {
        double v[2];
        int dst[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int e = e0 + u * nt;
            int i = int((sqrtf(8.0f * float(e) + 1.0f) - 1.0f) * 0.5f);
            if ((i + 1) * (i + 2) / 2 <= e) ++i;
            if (i * (i + 1) / 2 > e) --i;
            const int j = e - i * (i + 1) / 2;
            const int ic = i < n8 ? i : n8 - 1;       // e >= tot: discarded below
            const int jc = j < n8 ? j : 0;
            const double kv = kernel_value(kind, lam, dist2_exact(X[2 * ic], X[2 * ic + 1],
                                                                  X[2 * jc], X[2 * jc + 1]));
            double dg = xadd(1.0, NZ[ic]);
            if (jit != 0.0) dg = xadd(dg, jit);
            v[u] = i >= n ? (i == j ? 1.0 : 0.0) : (i == j ? dg : kv);
            dst[u] = e < tot ? CO[jc] + ic : -1;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
            if (dst[u] >= 0) L[dst[u]] = v[u];
    }
}

// A = K + diag(noise) (+ jitter) for one 8x8 tile (rows 8t.., block column
// kb) by one warp, two entries per lane (lane = row-major entry): the fill of
// block column kb+1 runs in the shadow of panel kb's factorisation chain.
__device__ __forceinline__ void warp_fill_tile(double* L, const int* CO, const double* X,
                                               const double* NZ, int n, int t, int kb, int kind,
                                               double lam, double jit, int lane) {
    double v[2];
    int dst[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int e = lane + 32 * u;
        const int i = 8 * t + (e >> 3), j = 8 * kb + (e & 7);
        const int ic = i < n ? i : 0, jc = j < n ? j : 0;
        const double kv = kernel_value(kind, lam, dist2_exact(X[2 * ic], X[2 * ic + 1],
                                                              X[2 * jc], X[2 * jc + 1]));
        double dg = xadd(1.0, NZ[ic]);
        if (jit != 0.0) dg = xadd(dg, jit);
        v[u] = (i >= n || j >= n) ? (i == j ? 1.0 : 0.0) : (i == j ? dg : kv);
        dst[u] = j <= i ? CO[j] + i : -1;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
        if (dst[u] >= 0) L[dst[u]] = v[u];
}

// Cholesky update of the 8x8 tile (rows 8t.., panel columns jp..jp+7):
// A -= L(rows, k_lo:k_hi) L(panel, k_lo:k_hi)^T with DMMA; k_lo, k_hi are
// multiples of 8 and the two k-chunks of each block column feed separate
// accumulators (half the dependent-DMMA chain); one CO lookup per block column.
__device__ __forceinline__ void chol_tile_update(double* L, const int* CO, int n8, int t, int jp,
                                                 int k_lo, int k_hi, int g, int tig) {
    const int rb = t * 8;
    double* p0 = L + CO[jp + 2 * tig] + rb + g;
    double* p1 = L + CO[jp + 2 * tig + 1] + rb + g;
    double c0 = *p0, c1 = *p1, d0 = 0.0, d1 = 0.0;
    for (int k8 = k_lo; k8 < k_hi; k8 += 8) {
        const double* col = L + CO[k8 + tig];
        const int o4 = 4 * tile_ldb(n8, k8 >> 3);
        dmma_acc(c0, c1, -col[rb + g], col[jp + g]);
        dmma_acc(d0, d1, -col[o4 + rb + g], col[o4 + jp + g]);
    }
    *p0 = c0 + d0;
    *p1 = c1 + d1;
}

// Step (b)+(c) of the panel Cholesky, run by each of `nft` threads: factor the
// 8x8 diagonal block at j0 in registers (dpotf2 order: scale by 1/sqrt(ajj),
// then the rank-1 update, gpr.py:187 cho_factor) - every thread redundantly,
// so there is no shuffle or shared-memory hand-off on the critical path - then
// solve this thread's row below the block, L(i, J) = A(i, J) L_JJ^-T, in the
// same operation order as the column-oriented substitution.  Thread 0
// publishes the factored block (LDG, row-major), 1/L_jj (INV) and the pivot
// flag (0 when a pivot is <= 0 or NaN, the dpotrf failure rule).
template <bool TWO>
__device__ __forceinline__ void chol_diag_and_rows(double* L, const int* CO, double* LDG,
                                                   double* INV, double* flag, int j0, int n8,
                                                   int tid, int nft) {
#ifdef VX_PHASE_TIMING
    long long tp = clock64();
#endif
    // block column j0/8 is column-major with leading dimension ldb from CO[j0]
    const int ldb = tile_ldb(n8, j0 >> 3);
    double* blk = L + CO[j0] + j0;                  // L(j0 + r, j0 + c) = blk[c * ldb + r]
    double a[36];                                   // packed lower triangle, row-major
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) a[r * (r + 1) / 2 + c] = blk[c * ldb + r];
#ifdef VX_PHASE_TIMING
    if (tid == 0) { const double s0 = a[35]; asm volatile("" :: "d"(s0)); }
#endif
    VX_PHASE(6, tp);                                // loads
    double inv[8];
    bool ok = true;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const double piv = a[c * (c + 1) / 2 + c];
        if (!(piv > 0.0)) ok = false;
        inv[c] = rsqrt(piv);
        a[c * (c + 1) / 2 + c] = piv * inv[c];
#pragma unroll
        for (int r = c + 1; r < 8; ++r) a[r * (r + 1) / 2 + c] *= inv[c];
#pragma unroll
        for (int r = c + 1; r < 8; ++r)
#pragma unroll
            for (int k = c + 1; k <= r; ++k)
                a[r * (r + 1) / 2 + k] = fma(-a[r * (r + 1) / 2 + c], a[k * (k + 1) / 2 + c],
                                             a[r * (r + 1) / 2 + k]);
    }
#ifdef VX_PHASE_TIMING
    if (tid == 0) { const double s1 = a[35] + inv[7]; asm volatile("" :: "d"(s1)); }
#endif
    VX_PHASE(7, tp);                                // factorisation chain
    VX_PHASE(8, tp);                                // (publish: after the rows)
    // TWO: two rows per thread per iteration (independent chains interleaved)
    for (int i = j0 + 8 + tid; i < n8; i += (TWO ? 2 : 1) * nft) {
        const bool two = TWO && i + nft < n8;
        double v[8], u[8];
        double* row = blk + (i - j0);
        double* row2 = row + (two ? nft : 0);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            v[c] = row[c * ldb];
            if (TWO) u[c] = row2[c * ldb];
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            v[c] *= inv[c];
            if (TWO) u[c] *= inv[c];
#pragma unroll
            for (int k = c + 1; k < 8; ++k) {
                v[k] = fma(-v[c], a[k * (k + 1) / 2 + c], v[k]);
                if (TWO) u[k] = fma(-u[c], a[k * (k + 1) / 2 + c], u[k]);
            }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) row[c * ldb] = v[c];
        if (two) {
#pragma unroll
            for (int c = 0; c < 8; ++c) row2[c * ldb] = u[c];
        }
    }
    // publish the factored block (lower part of LDG rows), 1/L_jj and the pivot
    // flag: static register indices by one thread, off the row-solve path
    if (tid == 0) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c <= r; ++c) LDG[(j0 + r) * 8 + c] = a[r * (r + 1) / 2 + c];
#pragma unroll
        for (int c = 0; c < 8; ++c) INV[j0 + c] = inv[c];
        *flag = ok ? 1.0 : 0.0;
    }
    VX_PHASE(9, tp);                                // rows below + publish
}

// ---------------------------------------------------------------------------
// CTA helpers shared by the DMMA tile and big kernels (voxel mode)
// ---------------------------------------------------------------------------
struct VoxelCtx {
    int s, vid, n, cnt, slot, axis;
    int64_t off;
    double mean_f, lo0, lo1, sp0, sp1;
};

// work item -> staged training set raw ∪ pseudo (voxel_map.py:196-200) split
// by the value axis: X (n, 2) parameter coordinates, F = f - mean(f)
// (gpr.py:291-294), NZ per-point noise; rows [n, npad) are zero.  Also the
// voxel's parameter-plane origin and extent (gpr.py:262-266).
__device__ __forceinline__ VoxelCtx team_stage_voxel(const VoxelSolveArgs& va, int it, double* X,
                                                     double* F, double* NZ, int npad, int tid,
                                                     int nt) {
    VoxelCtx c;
    c.s = va.items[it];
    c.vid = va.cand_voxel[c.s];
    c.n = va.cand_n[c.s];
    c.cnt = va.raw_count[c.vid];
    c.off = va.raw_offset[c.vid];
    c.slot = va.pred_slot[c.vid];
    c.axis = va.cand_axis[c.s];
    c.mean_f = va.cand_meanf[c.s];
    const int pa_ = param_axis_a(c.axis), pb_ = param_axis_b(c.axis);
    for (int r = tid; r < npad; r += nt) {
        if (r < c.n) {
            const double* p = train_point(va, r, c.cnt, c.off, c.slot);
            X[2 * r] = p[pa_];
            X[2 * r + 1] = p[pb_];
            F[r] = xsub(p[c.axis], c.mean_f);
            NZ[r] = r < c.cnt ? va.sensor_var : va.pred_var[int64_t(c.slot) * va.M + (r - c.cnt)];
        } else {
            X[2 * r] = X[2 * r + 1] = F[r] = NZ[r] = 0.0;
        }
    }
    c.lo0 = xmul(double(va.keys[int64_t(c.vid) * 3 + pa_]), va.voxel_size);
    c.lo1 = xmul(double(va.keys[int64_t(c.vid) * 3 + pb_]), va.voxel_size);
    c.sp0 = xsub(xadd(c.lo0, va.voxel_size), c.lo0);
    c.sp1 = xsub(xadd(c.lo1, va.voxel_size), c.lo1);
    return c;
}

// grid coordinates c_r = lo + ((r + 0.5) * (hi - lo)) / m (gpr.py:104-120):
// GC[r] on the first parameter axis, GC[mm + r] on the second
__device__ __forceinline__ void team_grid_coords(double* GC, const VoxelCtx& c, int mm, int tid) {
    if (tid < 2 * mm) {
        const int which = tid >= mm, r = tid - which * mm;
        GC[tid] = xadd(which ? c.lo1 : c.lo0, xdiv(xmul(double(r) + 0.5, which ? c.sp1 : c.sp0), double(mm)));
    }
}

// separable SE tables T[i * mm + r] = exp(-lam (x_i - c_r)^2), rows i < n:
// k*(x_i, (c_ri, c_si)) = EA[i][ri] * EB[i][si]
__device__ __forceinline__ void team_se_tables(double* EA, double* EB, const double* X,
                                               const double* GC, int n, int mm, double lam,
                                               int tid, int nt) {
    for (int e = tid; e < 2 * n; e += nt) {
        const int which = e >= n, i = e - which * n;
        const double xi = X[2 * i + which];
        const double* G = GC + which * mm;
        double* T = (which ? EB : EA) + i * mm;
#pragma unroll 3
        for (int r = 0; r < mm; ++r) {
            const double d = xsub(xi, G[r]);
            T[r] = exp(xmul(-lam, xmul(d, d)));
        }
    }
}

// column c of [f | K*] -> grid indices (ri, si) of query q = c - 1, packed
// ri | si << 16 (-1 for c == 0 and padding columns); query order is
// (sub-row, sub-col, fine-row, fine-col) as make_mesh_grid (gpr.py:104-120)
__device__ __forceinline__ void team_query_table(int* QT, const VoxelSolveArgs& va, int ncols_pad,
                                                 int tid, int nt) {
    for (int c = tid; c < ncols_pad; c += nt) {
        int v = -1;
        if (c >= 1 && c <= va.M) {
            const int q = c - 1;
            const int nr = va.n_r, ns = va.n_s, nr2 = nr * nr;
            const int sr = q / (ns * nr2);
            const int rem = q - sr * ns * nr2;
            const int sc = rem / nr2;
            const int rem2 = rem - sc * nr2;
            const int fr = rem2 / nr, fc = rem2 - fr * nr;
            v = (sr * nr + fr) | ((sc * nr + fc) << 16);
        }
        QT[c] = v;
    }
}

// Voxel epilogue (gpr.py:303-310, voxel_map.py:242-261): nearest training
// point in the parameter plane (first index on ties) with two threads per
// query, colour gather (all reads before any write: the colour source may be
// this voxel's previous prediction), assemble_points, clipped variances and
// the lifecycle update.  MU / VAR are indexed by column c = q + 1.
__device__ void team_voxel_epilogue(const VoxelSolveArgs& va, const VoxelCtx& c, const double* X,
                                    const double* GC, const int* QT, int mm, const double* MU,
                                    const double* VAR, double* COL, int tid, int nt) {
    const int m = va.M;
    const int h = (c.n + 1) >> 1;
    for (int t0 = 0; t0 < 2 * m; t0 += nt) {       // uniform trip count: pairs are lanes 2k, 2k+1
        const int t = t0 + tid, q = t >> 1, half = t & 1;
        double best = INFINITY;
        int bi = 0x7fffffff;
        if (q < m) {
            const int qt = QT[q + 1];
            const double g0 = GC[qt & 0xffff], g1 = GC[mm + (qt >> 16)];
            const int lo = half ? h : 0, hi = half ? c.n : h;
            for (int i = lo; i < hi; ++i) {
                const double d2 = dist2_exact(g0, g1, X[2 * i], X[2 * i + 1]);
                if (d2 < best) { best = d2; bi = i; }
            }
        }
        const double ob = __shfl_xor_sync(FULL, best, 1);
        const int oi = __shfl_xor_sync(FULL, bi, 1);
        if (ob < best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        if (q < m && half == 0) {
            if (bi >= c.n) bi = 0;
            const double* cs = bi < c.cnt ? va.raw_rgb + (c.off + bi) * 3
                                          : va.pred_rgb + (int64_t(c.slot) * m + (bi - c.cnt)) * 3;
            COL[q * 3] = cs[0];
            COL[q * 3 + 1] = cs[1];
            COL[q * 3 + 2] = cs[2];
        }
    }
    __syncthreads();
    const int pa_ = param_axis_a(c.axis);
    double* oxyz = va.pred_xyz + int64_t(c.slot) * m * 3;
    double* orgb = va.pred_rgb + int64_t(c.slot) * m * 3;
    double* ovar = va.pred_var + int64_t(c.slot) * m;
    for (int q = tid; q < m; q += nt) {
        // assemble_points (gpr.py:89-97)
        const int qt = QT[q + 1];
        const double pv = MU[q + 1], p0 = GC[qt & 0xffff], p1 = GC[mm + (qt >> 16)];
        oxyz[q * 3] = c.axis == 0 ? pv : (pa_ == 0 ? p0 : p1);
        oxyz[q * 3 + 1] = c.axis == 1 ? pv : (pa_ == 1 ? p0 : p1);
        oxyz[q * 3 + 2] = c.axis == 2 ? pv : (pa_ == 2 ? p0 : p1);
        orgb[q * 3] = COL[q * 3];
        orgb[q * 3 + 1] = COL[q * 3 + 1];
        orgb[q * 3 + 2] = COL[q * 3 + 2];
        ovar[q] = VAR[q + 1];
    }
    if (tid < 32) {
        const double mv = xdiv(warp_pairwise_sum(VAR + 1, m), double(m));
        if (tid == 0) {
            const uint8_t before = va.state[c.vid];
            const uint8_t after = mv <= va.eta ? VX_CONVERGED : VX_ACTIVE;
            va.state[c.vid] = after;
            va.value_axis[c.vid] = int8_t(c.axis);
            va.has_pred[c.vid] = 1;
            va.cand_status[c.s] = VX_ST_OK;
            va.cand_before[c.s] = before;
            va.cand_after[c.s] = after;
        }
    }
}

// Dynamic item queue of the persistent tile grids: a CTA's first item is
// blockIdx.x, later ones come from an atomic counter, so CTAs that drew small
// voxels take more of them (measured: the tile buckets 18.6 -> 18.2 ms vs the
// static blockIdx + k * gridDim stride).  Each launch takes its own counter
// from ONE library-wide ring (g_ctr_ring below, shared by every kernel
// instantiation), so two launches in flight on concurrent streams get different
// counters unless TILE_CTR_RING launches are issued while one is still running.
constexpr int TILE_CTR_RING = 4096;
__device__ int g_tile_ctr[TILE_CTR_RING];
static std::atomic<unsigned> g_ctr_ring{0};
static int next_queue_counter(int** ctr, cudaStream_t s) {
    VX_CUDA(cudaGetSymbolAddress(reinterpret_cast<void**>(ctr), g_tile_ctr));
    *ctr += g_ctr_ring.fetch_add(1) % TILE_CTR_RING;
    VX_CUDA(cudaMemsetAsync(*ctr, 0, sizeof(int), s));
    return VX_OK;
}
__device__ __forceinline__ int tile_next(int* s_next, int* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) *s_next = int(gridDim.x) + atomicAdd(ctr, 1);
    __syncthreads();
    return *s_next;
}
template <int NRB, int CTW, int NW, int MINB, int ROWS, bool VOXEL>
__global__ void __launch_bounds__(NW * 32, MINB) gpr_tile_kernel(VoxelSolveArgs va, ProblemArgs pa,
                                                           int mmax, int mm, int* ctr) {
    extern __shared__ __align__(16) double smem[];
    constexpr int N8 = NRB * 8;
    constexpr int NT = NW * 32;
    constexpr int PCOLS = NW * CTW * 8;             // right-hand sides per pass
    constexpr bool INC_FILL = NW >= 6;              // fill block columns in the chain's shadow
    const int MC = mmax + 1 > PCOLS ? mmax + 1 : PCOLS;   // columns of [f | K*] (padded)
    const TileLayout lay(N8, mm, MC, mmax, VOXEL);
    double* L = smem + lay.L;
    double* X = smem + lay.X;
    double* F = smem + lay.F;
    double* NZ = smem + lay.NZ;
    double* INV = smem + lay.INV;
    double* Z = smem + lay.Z;
    double* LDG = smem + lay.LDG;
    int* CO = reinterpret_cast<int*>(smem + lay.CO);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int num_items = VOXEL ? va.num_items : pa.num_items;
    double* GC = smem + lay.GC;
    int* QT = reinterpret_cast<int*>(smem + lay.QT);
    if constexpr (VOXEL) {
        team_query_table(QT, va, MC, tid, NT);
        __syncthreads();
    }

    __shared__ int s_next;
    for (int it = blockIdx.x; it < num_items; it = tile_next(&s_next, ctr)) {
#ifdef VX_PHASE_TIMING
        long long tph = clock64();
#endif
        int n, m, s, vid = 0, cnt = 0, slot = 0, axis = 2;
        int64_t off = 0, xo = 0, qo = 0;
        double lam, jitter, mean_f = 0.0;
        int kind;
        VoxelCtx vc{};
        if constexpr (VOXEL) {
            vc = team_stage_voxel(va, it, X, F, NZ, N8, tid, NT);
            s = vc.s;
            vid = vc.vid;
            n = vc.n;
            cnt = vc.cnt;
            off = vc.off;
            slot = vc.slot;
            axis = vc.axis;
            mean_f = vc.mean_f;
            m = va.M;
            lam = va.lam;
            jitter = va.jitter;
            kind = va.kernel;
            team_grid_coords(GC, vc, mm, tid);
            __syncthreads();
            if (kind == VX_KERNEL_SE) team_se_tables(smem + lay.EA, smem + lay.EB, X, GC, n, mm, lam, tid, NT);
        } else {
            s = pa.items[it];
            xo = pa.x_off[s];
            qo = pa.q_off[s];
            n = int(pa.x_off[s + 1] - xo);
            m = int(pa.q_off[s + 1] - qo);
            lam = pa.lam[s];
            jitter = pa.jitter;
            kind = pa.kernel;
            for (int r = tid; r < N8; r += NT) {
                if (r < n) {
                    X[2 * r] = pa.x[(xo + r) * 2];
                    X[2 * r + 1] = pa.x[(xo + r) * 2 + 1];
                    F[r] = pa.f[xo + r];
                    NZ[r] = pa.noise[xo + r];
                } else {
                    X[2 * r] = X[2 * r + 1] = F[r] = NZ[r] = 0.0;
                }
            }
        }
        const int nrb = (n + 7) >> 3;
        const int n8 = nrb * 8;
        for (int j = tid; j < n8; j += NT) {
            const int kb = j >> 3;
            int o = 0;
            for (int t = 0; t < kb; ++t) o += 8 * tile_ldb(n8, t);
            CO[j] = o + (j & 7) * tile_ldb(n8, kb) - 8 * kb;
        }
        __syncthreads();
        VX_PHASE(0, tph);                     // staging, grid, SE tables

        // ---- A (identity-padded), panel Cholesky with DMMA updates, one retry
        bool ok = false;
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            const double jit = attempt ? jitter : 0.0;
            // INC_FILL: block column 0 now; block column kb+1 is filled during
            // panel kb by the warps that do not factor (below), before their
            // look-ahead (measured: n > 64 buckets 6-7% faster; with 4 warps the
            // idle warps are too few and the up-front fill wins)
            if constexpr (INC_FILL)
                for (int t = warp; t < nrb; t += NW) warp_fill_tile(L, CO, X, NZ, n, t, 0, kind, lam, jit, lane);
            else
                team_fill_matrix(L, CO, X, NZ, n, n8, kind, lam, jit, tid, NT);
            __syncthreads();
            VX_PHASE(1, tph);                 // kernel matrix
            ok = true;
            // DMMA update of one 8x8 row tile of panel `jp` with columns [k_lo, k_hi)
            auto tile_update = [&](int t, int jp, int k_lo, int k_hi) {
                chol_tile_update(L, CO, n8, t, jp, k_lo, k_hi, g, tig);
            };
            bool la_prev = false;   // look-ahead already applied columns < j0 - 8 to this panel
#ifdef VX_PHASE_TIMING
            long long tsub = clock64();
#endif
            for (int kb = 0; kb < nrb; ++kb) {
                const int j0 = kb * 8;
                // (a) finish the panel update A(i, J) -= L(i, <j0) L(J, <j0)^T: after a
                // look-ahead only the previous panel's 8 columns remain
                if (j0 > 0) {
                    const int klo = la_prev ? j0 - 8 : 0;
                    for (int t = kb + warp; t < nrb; t += NW) tile_update(t, j0, klo, j0);
                    __syncthreads();
                }
                VX_PHASE(10, tsub);               // panel update + barrier
                // (b) every thread of the warps that own rows below this block (warp 0
                // at least) factors the 8x8 diagonal block in its own registers and
                // solves its row against it: no shuffles and no barrier between the
                // two.  The other warps meanwhile apply every final column (< j0) to
                // the NEXT panel (look-ahead), hiding the serial factorisation.
                const int below = n8 - j0 - 8;
                // ROWS = 2: the factor warps solve two rows per thread, so more
                // warps are free for the fill and look-ahead of the next block
                // column (balances the two paths of a panel for n > 96)
                int nfw = ROWS == 2 ? (below > 64 ? (below + 63) / 64 : 1) : (below > 32 ? (below + 31) / 32 : 1);
                if (nfw >= NW) nfw = NW - 1;          // keep a warp for the fill of the next block column
                const bool la = (kb + 1 < nrb) && (NW > nfw) && j0 > 0;
                if (warp >= nfw) {
                    for (int t = kb + 1 + (warp - nfw); t < nrb; t += NW - nfw) {
                        if constexpr (INC_FILL) {
                            warp_fill_tile(L, CO, X, NZ, n, t, kb + 1, kind, lam, jit, lane);
                            __syncwarp();
                        }
                        if (la) tile_update(t, j0 + 8, 0, j0);
                    }
                } else {
                    chol_diag_and_rows<ROWS == 2>(L, CO, LDG, INV, smem + lay.FLAG, j0, n8, tid, (nfw < NW ? nfw : NW) * 32);
                }
#ifdef VX_PHASE_TIMING
                tsub = clock64();
#endif
                __syncthreads();
                VX_PHASE(11, tsub);               // barrier after the factorisation
                la_prev = la;
                if (smem[lay.FLAG] == 0.0) {          // pivot <= 0 or NaN: uniform exit
                    ok = false;
                    break;
                }
            }
            __syncthreads();
        }
        VX_PHASE(2, tph);                     // panel Cholesky
        if (!ok) {
            if (tid == 0) {
                if constexpr (VOXEL) {
                    va.cand_status[s] = VX_ST_CHOL_FAIL;
                    const uint8_t st = va.state[vid];
                    va.cand_before[s] = st;
                    va.cand_after[s] = st;
                } else {
                    pa.status[s] = VX_ST_CHOL_FAIL;
                }
            }
            __syncthreads();
            continue;
        }
        // inverses of the diagonal blocks (thread = (block, column)): L_kk x = e_c
        double* LINV = smem + lay.LINV;
        // (LINV overlays LDG: every block is read before any thread overwrites it)
        for (int t0 = 0; t0 < nrb * 8; t0 += NT) {
            const int t = t0 + tid;
            const int kb = t >> 3, c = t & 7, b0 = kb * 8;
            double x[8];
            if (t < nrb * 8) {
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    double v = (r == c) ? 1.0 : 0.0;
#pragma unroll
                    for (int k = 0; k < r; ++k) v = fma(-LDG[(b0 + r) * 8 + k], x[k], v);
                    x[r] = (r < c) ? 0.0 : v * INV[b0 + r];
                }
            }
            __syncthreads();
            if (t < nrb * 8) {
#pragma unroll
                for (int r = 0; r < 8; ++r) LINV[(b0 + r) * 8 + c] = x[r];
            }
        }
        __syncthreads();

        VX_PHASE(3, tph);                     // diagonal-block inverses
        // ---- forward substitution: right-hand sides resident as DMMA accumulators
        const int ncols = m + 1;
        const double* EA = smem + lay.EA;
        const double* EB = smem + lay.EB;
        for (int c0 = 0; c0 < ncols; c0 += PCOLS) {
            double C[NRB][CTW][2];
            // right-hand side values: rows 8 rb + g, columns c0 + 8 (warp*CTW + ct) + 2 tig + e
#pragma unroll
            for (int ct = 0; ct < CTW; ++ct) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = c0 + (warp * CTW + ct) * 8 + 2 * tig + e;
                    const int q = c - 1;
                    int ri = 0, si = 0;
                    double g0 = 0, g1 = 0;
                    if (c > 0 && c < ncols) {
                        if constexpr (VOXEL) {
                            const int qt = QT[c];
                            ri = qt & 0xffff;
                            si = qt >> 16;
                            g0 = GC[ri];
                            g1 = GC[mm + si];
                        } else {
                            g0 = pa.xs[(qo + q) * 2];
                            g1 = pa.xs[(qo + q) * 2 + 1];
                        }
                    }
#pragma unroll
                    for (int rb = 0; rb < NRB; ++rb) {
                        const int i = rb * 8 + g;
                        double v = 0.0;
                        if (rb < nrb && i < n && c < ncols) {
                            if (c == 0) v = F[i];
                            else if (VOXEL && kind == VX_KERNEL_SE) v = EA[i * mm + ri] * EB[i * mm + si];
                            else v = kernel_value(kind, lam, dist2_exact(X[2 * i], X[2 * i + 1], g0, g1));
                        }
                        C[rb][ct][e] = v;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < NRB; ++k) {
                if (k < nrb) {
                    // diagonal block: W_k = L_kk^-1 C_k with DMMA (C_k -> B fragments by shuffles)
                    {
                        double bc[CTW][2];
#pragma unroll
                        for (int ct = 0; ct < CTW; ++ct) {
#pragma unroll
                            for (int sl = 0; sl < 2; ++sl) {
                                const int src = (4 * sl + tig) * 4 + (g >> 1);
                                const double v0 = __shfl_sync(FULL, C[k][ct][0], src);
                                const double v1 = __shfl_sync(FULL, C[k][ct][1], src);
                                bc[ct][sl] = (g & 1) ? v1 : v0;
                            }
                        }
                        const double a0 = LINV[(k * 8 + g) * 8 + tig];
                        const double a1 = LINV[(k * 8 + g) * 8 + 4 + tig];
#pragma unroll
                        for (int ct = 0; ct < CTW; ++ct) {
                            double d0 = 0.0, d1 = 0.0;
                            dmma_acc(d0, d1, a0, bc[ct][0]);
                            dmma_acc(d0, d1, a1, bc[ct][1]);
                            C[k][ct][0] = d0;
                            C[k][ct][1] = d1;
                        }
                    }
                    if (k + 1 < nrb) {
                        // W_k as B fragments: B_s[tig][g] = W(8k + 4s + tig, col 8ct + g)
                        double bf[CTW][2];
#pragma unroll
                        for (int ct = 0; ct < CTW; ++ct) {
#pragma unroll
                            for (int sl = 0; sl < 2; ++sl) {
                                const int src = (4 * sl + tig) * 4 + (g >> 1);
                                const double v0 = __shfl_sync(FULL, C[k][ct][0], src);
                                const double v1 = __shfl_sync(FULL, C[k][ct][1], src);
                                bf[ct][sl] = (g & 1) ? v1 : v0;
                            }
                        }
#pragma unroll
                        for (int k2 = k + 1; k2 < NRB; ++k2) {
                            if (k2 < nrb) {
#pragma unroll
                                for (int sl = 0; sl < 2; ++sl) {
                                    const double a = -L[CO[k * 8 + 4 * sl + tig] + k2 * 8 + g];
#pragma unroll
                                    for (int ct = 0; ct < CTW; ++ct)
                                        dmma_acc(C[k2][ct][0], C[k2][ct][1], a, bf[ct][sl]);
                                }
                            }
                        }
                    }
                }
            }
            // z = L^-1 f (global column 0) to shared memory
            if (c0 == 0 && warp == 0 && tig == 0) {
#pragma unroll
                for (int rb = 0; rb < NRB; ++rb)
                    if (rb < nrb) Z[rb * 8 + g] = C[rb][0][0];
            }
            __syncthreads();
            // per-column sum of squares and mu = w . z, reduced over the row groups g
#pragma unroll
            for (int ct = 0; ct < CTW; ++ct) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    double ss = 0.0, mu = 0.0;
#pragma unroll
                    for (int rb = 0; rb < NRB; ++rb) {
                        if (rb < nrb) {
                            const double w = C[rb][ct][e];
                            ss = fma(w, w, ss);
                            mu = fma(w, Z[rb * 8 + g], mu);
                        }
                    }
#pragma unroll
                    for (int o = 4; o < 32; o <<= 1) {
                        ss += __shfl_xor_sync(FULL, ss, o);
                        mu += __shfl_xor_sync(FULL, mu, o);
                    }
                    const int lc = (warp * CTW + ct) * 8 + 2 * tig + e;   // column within the pass
                    const int c = c0 + lc;
                    if (g == 0 && c > 0 && c < ncols) {
                        const double var = 1.0 - ss;
                        if constexpr (VOXEL) {
                            smem[lay.MU + c] = xadd(mu, mean_f);      // by global column
                            smem[lay.VAR + c] = var < 0.0 ? 0.0 : var;
                        } else {
                            pa.mu[qo + c - 1] = mu;
                            pa.var[qo + c - 1] = var;
                        }
                    }
                }
            }
            __syncthreads();
        }
        if constexpr (VOXEL) {
            // every pass has written MU / VAR (indexed by column): epilogue once
            VX_PHASE(4, tph);                 // forward substitution + reductions
            team_voxel_epilogue(va, vc, X, GC, QT, mm, smem + lay.MU, smem + lay.VAR,
                                smem + lay.COL, tid, NT);
        }
        if constexpr (!VOXEL) {
            if (tid == 0) pa.status[s] = VX_ST_OK;
        }
        __syncthreads();
        VX_PHASE(5, tph);                     // epilogue
    }
}

template <int NW, bool VOXEL, bool SMEM>
__global__ void __launch_bounds__(NW * 32, NW <= 6 ? 2 : 1) gpr_big_kernel(
        VoxelSolveArgs va, ProblemArgs pa, int mmax, int mm, int nmax, double* gwork,
        int64_t per_cta) {
    // SMEM: everything but W in dynamic shared memory, W in a per-CTA global
    // slice; otherwise every buffer lives in the per-CTA global workspace.
    extern __shared__ __align__(16) double dsm[];
    constexpr int CTW = 1;
    constexpr int NT = NW * 32;
    constexpr int PCOLS = NW * CTW * 8;             // right-hand sides per pass
    const int N8 = ((nmax + 7) / 8) * 8;
    const int MC = (mmax + 1 > PCOLS ? mmax + 1 : PCOLS);
    const TileLayout lay(N8, mm, MC, mmax, VOXEL, !SMEM);
    double* smem = SMEM ? dsm : gwork + int64_t(blockIdx.x) * per_cta;
    double* Wg = SMEM ? gwork + int64_t(blockIdx.x) * per_cta : smem + lay.W;
    double* L = smem + lay.L;
    double* X = smem + lay.X;
    double* F = smem + lay.F;
    double* NZ = smem + lay.NZ;
    double* INV = smem + lay.INV;
    double* Z = smem + lay.Z;
    double* LDG = smem + lay.LDG;
    int* CO = reinterpret_cast<int*>(smem + lay.CO);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int num_items = VOXEL ? va.num_items : pa.num_items;
    double* GC = smem + lay.GC;
    int* QT = reinterpret_cast<int*>(smem + lay.QT);
    if constexpr (VOXEL) {
        team_query_table(QT, va, MC, tid, NT);
        __syncthreads();
    }

    for (int it = blockIdx.x; it < num_items; it += gridDim.x) {
        int n, m, s, vid = 0, cnt = 0, slot = 0, axis = 2;
        int64_t off = 0, xo = 0, qo = 0;
        double lam, jitter, mean_f = 0.0;
        int kind;
        VoxelCtx vc{};
        if constexpr (VOXEL) {
            vc = team_stage_voxel(va, it, X, F, NZ, N8, tid, NT);
            s = vc.s;
            vid = vc.vid;
            n = vc.n;
            cnt = vc.cnt;
            off = vc.off;
            slot = vc.slot;
            axis = vc.axis;
            mean_f = vc.mean_f;
            m = va.M;
            lam = va.lam;
            jitter = va.jitter;
            kind = va.kernel;
            team_grid_coords(GC, vc, mm, tid);
            __syncthreads();
            if (kind == VX_KERNEL_SE) team_se_tables(smem + lay.EA, smem + lay.EB, X, GC, n, mm, lam, tid, NT);
        } else {
            s = pa.items[it];
            xo = pa.x_off[s];
            qo = pa.q_off[s];
            n = int(pa.x_off[s + 1] - xo);
            m = int(pa.q_off[s + 1] - qo);
            lam = pa.lam[s];
            jitter = pa.jitter;
            kind = pa.kernel;
            for (int r = tid; r < N8; r += NT) {
                if (r < n) {
                    X[2 * r] = pa.x[(xo + r) * 2];
                    X[2 * r + 1] = pa.x[(xo + r) * 2 + 1];
                    F[r] = pa.f[xo + r];
                    NZ[r] = pa.noise[xo + r];
                } else {
                    X[2 * r] = X[2 * r + 1] = F[r] = NZ[r] = 0.0;
                }
            }
        }
        const int nrb = (n + 7) >> 3;
        const int n8 = nrb * 8;
        for (int j = tid; j < n8; j += NT) {
            const int kb = j >> 3;
            int o = 0;
            for (int t = 0; t < kb; ++t) o += 8 * tile_ldb(n8, t);
            CO[j] = o + (j & 7) * tile_ldb(n8, kb) - 8 * kb;
        }
        __syncthreads();

        // ---- A (identity-padded), panel Cholesky with DMMA updates, one retry
        bool ok = false;
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            const double jit = attempt ? jitter : 0.0;
            // shared-memory variant (n <= ~160): block column 0 now, block column
            // kb+1 during panel kb (as the tile kernel); larger n fill up front
            // (too few idle warps next to the long early panels)
            if constexpr (SMEM)
                for (int t = warp; t < nrb; t += NW) warp_fill_tile(L, CO, X, NZ, n, t, 0, kind, lam, jit, lane);
            else
                team_fill_matrix(L, CO, X, NZ, n, n8, kind, lam, jit, tid, NT);
            __syncthreads();
            ok = true;
            // DMMA update of one 8x8 row tile of panel `jp` with columns [k_lo, k_hi)
            auto tile_update = [&](int t, int jp, int k_lo, int k_hi) {
                chol_tile_update(L, CO, n8, t, jp, k_lo, k_hi, g, tig);
            };
            bool la_prev = false;   // look-ahead already applied columns < j0 - 8 to this panel
            for (int kb = 0; kb < nrb; ++kb) {
                const int j0 = kb * 8;
                // (a) finish the panel update A(i, J) -= L(i, <j0) L(J, <j0)^T: after a
                // look-ahead only the previous panel's 8 columns remain
                if (j0 > 0) {
                    const int klo = la_prev ? j0 - 8 : 0;
                    for (int t = kb + warp; t < nrb; t += NW) tile_update(t, j0, klo, j0);
                    __syncthreads();
                }
                // (b) every thread of the warps that own rows below this block (warp 0
                // at least) factors the 8x8 diagonal block in its own registers and
                // solves its row against it: no shuffles and no barrier between the
                // two.  The other warps meanwhile apply every final column (< j0) to
                // the NEXT panel (look-ahead), hiding the serial factorisation.
                const int below = n8 - j0 - 8;
                int nfw = below > 32 ? (below + 31) / 32 : 1;
                if (SMEM && nfw >= NW) nfw = NW - 1;  // keep a warp for the fill of the next block column
                const bool la = (kb + 1 < nrb) && (NW > nfw) && j0 > 0;
                if (warp >= nfw) {
                    for (int t = kb + 1 + (warp - nfw); t < nrb; t += NW - nfw) {
                        if constexpr (SMEM) {
                            warp_fill_tile(L, CO, X, NZ, n, t, kb + 1, kind, lam, jit, lane);
                            __syncwarp();
                        }
                        if (la) tile_update(t, j0 + 8, 0, j0);
                    }
                } else {
                    chol_diag_and_rows<false>(L, CO, LDG, INV, smem + lay.FLAG, j0, n8, tid, (nfw < NW ? nfw : NW) * 32);
                }
                __syncthreads();
                la_prev = la;
                if (smem[lay.FLAG] == 0.0) {          // pivot <= 0 or NaN: uniform exit
                    ok = false;
                    break;
                }
            }
            __syncthreads();
        }
        if (!ok) {
            if (tid == 0) {
                if constexpr (VOXEL) {
                    va.cand_status[s] = VX_ST_CHOL_FAIL;
                    const uint8_t st = va.state[vid];
                    va.cand_before[s] = st;
                    va.cand_after[s] = st;
                } else {
                    pa.status[s] = VX_ST_CHOL_FAIL;
                }
            }
            __syncthreads();
            continue;
        }
        // inverses of the diagonal blocks (thread = (block, column)): L_kk x = e_c
        double* LINV = smem + lay.LINV;
        // (LINV overlays LDG: every block is read before any thread overwrites it)
        for (int t0 = 0; t0 < nrb * 8; t0 += NT) {
            const int t = t0 + tid;
            const int kb = t >> 3, c = t & 7, b0 = kb * 8;
            double x[8];
            if (t < nrb * 8) {
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    double v = (r == c) ? 1.0 : 0.0;
#pragma unroll
                    for (int k = 0; k < r; ++k) v = fma(-LDG[(b0 + r) * 8 + k], x[k], v);
                    x[r] = (r < c) ? 0.0 : v * INV[b0 + r];
                }
            }
            __syncthreads();
            if (t < nrb * 8) {
#pragma unroll
                for (int r = 0; r < 8; ++r) LINV[(b0 + r) * 8 + c] = x[r];
            }
        }
        __syncthreads();

        // ---- forward substitution, left-looking: C_k = B_k - sum_j L_kj W_j by DMMA
        // (two accumulator chains), W_k = L_kk^-1 C_k, W kept row-major in the workspace
        const int ncols = m + 1;
        const double* EA = smem + lay.EA;
        const double* EB = smem + lay.EB;
        for (int c0 = 0; c0 < ncols; c0 += PCOLS) {
            const int ctile = warp;                       // one 8-column tile per warp
            int ri[2] = {0, 0}, si[2] = {0, 0};
            double g0[2] = {0, 0}, g1[2] = {0, 0};
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = c0 + ctile * 8 + 2 * tig + e;
                const int q = c - 1;
                if (c > 0 && c < ncols) {
                    if constexpr (VOXEL) {
                        const int qt = QT[c];
                        ri[e] = qt & 0xffff;
                        si[e] = qt >> 16;
                        g0[e] = GC[ri[e]];
                        g1[e] = GC[mm + si[e]];
                    } else {
                        g0[e] = pa.xs[(qo + q) * 2];
                        g1[e] = pa.xs[(qo + q) * 2 + 1];
                    }
                }
            }
            double ssp[2] = {0.0, 0.0};
            for (int k = 0; k < nrb; ++k) {
                double ca[2], cb[2] = {0.0, 0.0};
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = c0 + ctile * 8 + 2 * tig + e;
                    const int i = k * 8 + g;
                    double v = 0.0;
                    if (i < n && c < ncols) {
                        if (c == 0) v = F[i];
                        else if (VOXEL && kind == VX_KERNEL_SE) v = EA[i * mm + ri[e]] * EB[i * mm + si[e]];
                        else v = kernel_value(kind, lam, dist2_exact(X[2 * i], X[2 * i + 1], g0[e], g1[e]));
                    }
                    ca[e] = v;
                }
                for (int j = 0; j < k; ++j) {
#pragma unroll
                    for (int sl = 0; sl < 2; ++sl) {
                        const int kk = j * 8 + 4 * sl + tig;
                        const double a = -L[CO[kk] + k * 8 + g];
                        const double bw = Wg[int64_t(kk) * PCOLS + ctile * 8 + g];
                        if (sl == 0) dmma_acc(ca[0], ca[1], a, bw);
                        else dmma_acc(cb[0], cb[1], a, bw);
                    }
                }
                ca[0] += cb[0];
                ca[1] += cb[1];
                // W_k = L_kk^-1 C_k (C_k -> B fragments by shuffles)
                double bc[2];
#pragma unroll
                for (int sl = 0; sl < 2; ++sl) {
                    const int src = (4 * sl + tig) * 4 + (g >> 1);
                    const double v0 = __shfl_sync(FULL, ca[0], src);
                    const double v1 = __shfl_sync(FULL, ca[1], src);
                    bc[sl] = (g & 1) ? v1 : v0;
                }
                double d0 = 0.0, d1 = 0.0;
                dmma_acc(d0, d1, LINV[(k * 8 + g) * 8 + tig], bc[0]);
                dmma_acc(d0, d1, LINV[(k * 8 + g) * 8 + 4 + tig], bc[1]);
                Wg[int64_t(k * 8 + g) * PCOLS + ctile * 8 + 2 * tig] = d0;
                Wg[int64_t(k * 8 + g) * PCOLS + ctile * 8 + 2 * tig + 1] = d1;
                ssp[0] = fma(d0, d0, ssp[0]);
                ssp[1] = fma(d1, d1, ssp[1]);
                __syncwarp();
            }
            __syncthreads();
            if (c0 == 0)
                for (int i = tid; i < n8; i += NT) Z[i] = Wg[int64_t(i) * PCOLS];   // z = L^-1 f
            __syncthreads();
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double ss = ssp[e], mu = 0.0;
                for (int k = 0; k < nrb; ++k)
                    mu = fma(Wg[int64_t(k * 8 + g) * PCOLS + ctile * 8 + 2 * tig + e], Z[k * 8 + g], mu);
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) {
                    ss += __shfl_xor_sync(FULL, ss, o);
                    mu += __shfl_xor_sync(FULL, mu, o);
                }
                const int lc = ctile * 8 + 2 * tig + e;
                const int c = c0 + lc;
                if (g == 0 && c > 0 && c < ncols) {
                    const double var = 1.0 - ss;
                    if constexpr (VOXEL) {
                        smem[lay.MU + c] = xadd(mu, mean_f);
                        smem[lay.VAR + c] = var < 0.0 ? 0.0 : var;
                    } else {
                        pa.mu[qo + c - 1] = mu;
                        pa.var[qo + c - 1] = var;
                    }
                }
            }
            __syncthreads();
        }
        {
            if constexpr (VOXEL) {
                // every pass has written MU / VAR (indexed by column): epilogue once
                __syncthreads();
                team_voxel_epilogue(va, vc, X, GC, QT, mm, smem + lay.MU, smem + lay.VAR,
                                    smem + lay.COL, tid, NT);
            }
            __syncthreads();
        }
        if constexpr (!VOXEL) {
            if (tid == 0) pa.status[s] = VX_ST_OK;
        }
        __syncthreads();
    }
}

#include "vx_panel.cuh"

// tile-kernel configurations per size bucket: (8-column tiles per warp and
// pass, warps per CTA, resident CTAs per SM the registers are capped for,
// rows per factor thread in the panel solve)
#ifndef T64_CTW
#define T64_CTW 1             // four 4-warp CTAs per SM (measured: 4.55 -> 4.02 ms vs two 6-warp CTAs)
#define T64_NW 4
#define T64_MINB 4
#define T64_ROWS 1
#endif
#ifndef T96_NRB
#define T96_NRB 12            // own 96-row instantiation (measured: 6.22 -> 6.07 ms vs the 128-row kernel)
#define T96_CTW 1
#define T96_NW 6
#define T96_MINB 2
#define T96_ROWS 1
#endif
#ifndef T128_CTW
#define T128_CTW 1
#define T128_NW 6
#define T128_MINB 2
#define T128_ROWS 2           // two rows per factor thread (measured: 8.60 -> 8.29 ms)
#endif
#ifndef T160_NW
#define T160_NW 12
#define T160_ROWS 1
#endif
#define T64_CFG T64_CTW, T64_NW, T64_MINB, T64_ROWS
#define T96_CFG T96_CTW, T96_NW, T96_MINB, T96_ROWS
#define T128_CFG T128_CTW, T128_NW, T128_MINB, T128_ROWS

template <int NRB, int CTW, int NW, int MINB, int ROWS, bool VOXEL>
static int launch_tile(const VoxelSolveArgs& va, const ProblemArgs& pa, int num_items, int m_max,
                       int mm, cudaStream_t s) {
    if (num_items <= 0) return VX_OK;
    constexpr int PCOLS = NW * CTW * 8;
    const int MC = m_max + 1 > PCOLS ? m_max + 1 : PCOLS;
    const TileLayout lay(NRB * 8, mm, MC, m_max, VOXEL);
    const size_t smem = size_t(lay.total) * sizeof(double);
    auto kfn = gpr_tile_kernel<NRB, CTW, NW, MINB, ROWS, VOXEL>;
    VX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;       // resident CTAs (registers and shared memory): the grid is persistent
    VX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, NW * 32, smem));
    if (per_sm < 1) per_sm = 1;
#ifdef VX_PHASE_TIMING
    if (getenv("VX_TILE_PER_SM")) per_sm = atoi(getenv("VX_TILE_PER_SM"));
#endif
    int blocks = num_items;
    const int cap = sm_count() * per_sm;
    if (blocks > cap) blocks = cap;
    int* ctr = nullptr;
    VX_TRY(next_queue_counter(&ctr, s));
    kfn<<<blocks, NW * 32, smem, s>>>(va, pa, m_max, mm, ctr);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}


// Items of the large-n bucket sorted by n, largest first (one CTA: counting
// sort over n in [lo, lo + 4096); order within one n is arbitrary, which does
// not matter: every item's result is independent of the others).
template <bool VOXEL>
__global__ void __launch_bounds__(1024) k_sort_items_desc(VoxelSolveArgs va, ProblemArgs pa, int count,
                                                          int hi, int32_t* out) {
    __shared__ int hist[4096];
    const int* items = VOXEL ? va.items : pa.items;
    auto key = [&](int i) {
        const int s = items[i];
        const int n = VOXEL ? va.cand_n[s] : int(pa.x_off[s + 1] - pa.x_off[s]);
        int b = hi - n;                       // largest n -> bin 0
        return b < 0 ? 0 : (b > 4095 ? 4095 : b);
    };
    for (int b = threadIdx.x; b < 4096; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < count; i += blockDim.x) atomicAdd(&hist[key(i)], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int b = 0; b < 4096; ++b) {
            const int c = hist[b];
            hist[b] = acc;
            acc += c;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < count; i += blockDim.x) out[atomicAdd(&hist[key(i)], 1)] = items[i];
}

// Team size (CTAs per cluster) of the panel kernel: few items -> spread each
// voxel over up to 8 SMs (latency, e.g. one Livox scan); many items -> one CTA
// per voxel.  VX_PANEL_C overrides (A/B experiments).
static int panel_team_size(int num_items) {
    if (const char* e = getenv("VX_PANEL_C")) {
        const int c = atoi(e);
        if (c == 1 || c == 2 || c == 4 || c == 8 || c == 16) return c;
    }
    // up to two rounds of the team count: the largest voxel (first in the
    // queue) sets the latency, so bigger teams win (config 3: ~30 items)
    const int sms = sm_count();
    if (num_items * 4 <= sms) return 8;
    if (num_items * 2 <= sms) return 4;
    if (num_items <= sms) return 2;
    return 1;
}

template <bool VOXEL>
static int launch_panel(const VoxelSolveArgs& va_in, const ProblemArgs& pa_in, int num_items,
                        int n_max, int m_max, int mm, DevBuf& work, cudaStream_t s) {
    if (num_items <= 0) return VX_OK;
    VoxelSolveArgs va = va_in;
    ProblemArgs pa = pa_in;
    const int C = panel_team_size(num_items);
    const int NP = round_up(n_max, PNB);
    const int A32 = round_up(m_max + 1, PNB);
    const int R = NP + A32;
    const int MC = m_max + 1 > 96 ? round_up(m_max + 1, 32) : 96;
    const PanelLayout lay(NP, MC, m_max);
    const size_t smem = size_t(lay.total) * sizeof(double);
    auto kfn = gpr_panel_kernel<VOXEL>;
    VX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (C > 8) VX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int per_sm = 1;
    VX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, PNT, smem));
    if (per_sm < 1) per_sm = 1;
    int teams = (sm_count() * per_sm) / C;
    if (teams > num_items) teams = num_items;
    if (teams < 1) teams = 1;
    PanelArgs pk{};
    pk.per_team = panel_base(R, NP / PNB);
    pk.partial_per_team = int64_t(C) * PW * 2 * A32;
    pk.csize = C;
    pk.nmax = n_max;
    pk.mmax = m_max;
    pk.mm = mm;
    // workspace: sorted items | team slots | partial sums | L panels
    const size_t items_b = (size_t(num_items) * 4 + 255) & ~size_t(255);
    const size_t slots_b = (size_t(teams) * 4 + 255) & ~size_t(255);
    const size_t part_b = size_t(teams) * pk.partial_per_team * 8;
    const size_t l_b = size_t(teams) * pk.per_team * 8;
    VX_TRY(work.reserve(items_b + slots_b + part_b + l_b, s));
    char* base = work.as<char>();
    int32_t* sorted = reinterpret_cast<int32_t*>(base);
    pk.slots = reinterpret_cast<int*>(base + items_b);
    pk.partial = reinterpret_cast<double*>(base + items_b + slots_b);
    pk.work = reinterpret_cast<double*>(base + items_b + slots_b + part_b);
    k_sort_items_desc<VOXEL><<<1, 1024, 0, s>>>(va, pa, num_items, n_max, sorted);
    count_launch();
    VX_CHECK_LAUNCH();
    if (VOXEL) va.items = sorted; else pa.items = sorted;
    VX_TRY(next_queue_counter(&pk.queue, s));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(teams * C));
    cfg.blockDim = dim3(PNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    VX_CUDA(cudaLaunchKernelEx(&cfg, kfn, va, pa, pk));
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

template <int NW, bool VOXEL>
static int launch_big(const VoxelSolveArgs& va, const ProblemArgs& pa, int num_items, int n_max,
                      int m_max, int mm, DevBuf& work, cudaStream_t s) {
    if (num_items <= 0) return VX_OK;
    constexpr int PCOLS = NW * 8;
    const int n8 = ((n_max + 7) / 8) * 8;
    const int MC = m_max + 1 > PCOLS ? m_max + 1 : PCOLS;
    // shared-memory variant when everything but W fits two CTAs per SM
    const TileLayout small(n8, mm, MC, m_max, VOXEL, false);
    const size_t smem = size_t(small.total) * sizeof(double);
    const bool use_smem = smem <= size_t(NW <= 6 ? 112 : 220) * 1024;
    const TileLayout full(n8, mm, MC, m_max, VOXEL, true);
    const int64_t per = use_smem ? int64_t(n8) * PCOLS : full.total;
    int blocks = num_items;
    // persistent grid: resident CTAs only (a CTA beyond residency would start
    // its strided share of the items after a whole resident CTA finished)
    int per_sm = 2;
    if (use_smem) {
        VX_CUDA(cudaFuncSetAttribute(gpr_big_kernel<NW, VOXEL, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        VX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gpr_big_kernel<NW, VOXEL, true>,
                                                              NW * 32, smem));
    } else {
        VX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gpr_big_kernel<NW, VOXEL, false>,
                                                              NW * 32, 0));
    }
    if (per_sm < 1) per_sm = 1;
    int cap = sm_count() * per_sm;
    const int64_t max_blocks = (int64_t(4) << 30) / (per * 8);
    if (cap > max_blocks) cap = int(max_blocks > 0 ? max_blocks : 1);
    if (blocks > cap) blocks = cap;
    VX_TRY(work.reserve(size_t(per) * 8 * blocks, s));
    if (use_smem) {
        auto kfn = gpr_big_kernel<NW, VOXEL, true>;
        kfn<<<blocks, NW * 32, smem, s>>>(va, pa, m_max, mm, n_max, work.as<double>(), per);
    } else {
        gpr_big_kernel<NW, VOXEL, false><<<blocks, NW * 32, 0, s>>>(va, pa, m_max, mm, n_max,
                                                                    work.as<double>(), per);
    }
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

template <bool VOXEL>
static int launch_cta(const VoxelSolveArgs& va, const ProblemArgs& pa, int num_items, int n_max,
                      int m_max, int mm, DevBuf& work, cudaStream_t s) {
    if (num_items <= 0) return VX_OK;
    const CtaLayout lay(n_max, mm, m_max, VOXEL);
    const size_t bytes = size_t(lay.total) * sizeof(double);
    auto kfn = gpr_cta_kernel<VOXEL>;
    int blocks = num_items;
    double* gw = nullptr;
    size_t smem = 0;
    if (bytes <= size_t(220) * 1024) {
        smem = bytes;
        VX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int per_sm = int((size_t(227) * 1024) / (smem + 1024));
        if (per_sm < 1) per_sm = 1;
        if (per_sm > 8) per_sm = 8;
        const int cap = sm_count() * per_sm;
        if (blocks > cap) blocks = cap;
    } else {
        int cap = sm_count() * 6;      // latency-bound on the L2 workspace: oversubscribe
        const int64_t max_blocks = (int64_t(4) << 30) / int64_t(bytes);
        if (cap > max_blocks) cap = int(max_blocks > 0 ? max_blocks : 1);
        if (blocks > cap) blocks = cap;
        VX_TRY(work.reserve(bytes * blocks, s));
        gw = work.as<double>();
    }
    kfn<<<blocks, CT, smem, s>>>(va, pa, n_max, m_max, mm, gw, int64_t(lay.total));
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
template <int NMAX, bool VOXEL>
static int launch_warp(const VoxelSolveArgs& va, const ProblemArgs& pa, int num_items, int m_max,
                       int mm, cudaStream_t s) {
    if (num_items <= 0) return VX_OK;
    const WarpLayout lay(NMAX, mm, m_max, VOXEL);
    const size_t per_warp = size_t(lay.total) * sizeof(double);
    int wpb = 4;
    while (wpb > 1 && per_warp * wpb > size_t(100) * 1024) --wpb;
    const size_t smem = per_warp * wpb;
    auto kfn = gpr_warp_kernel<NMAX, VOXEL>;
    VX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int blocks = (num_items + wpb - 1) / wpb;
    const int cap = sm_count() * 16;
    if (blocks > cap) blocks = cap;
    kfn<<<blocks, 32 * wpb, smem, s>>>(va, pa, m_max, mm);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

template <int NMAX>
static int launch_wdmma(const VoxelSolveArgs& va, int mm, cudaStream_t s) {
    if (va.num_items <= 0) return VX_OK;
    const WarpLayout lay(NMAX, mm, va.M, true);
    const int ntiles = (va.M + 1 + 7) / 8;
    constexpr int wpb = 4;
    const size_t smem = size_t(lay.total) * sizeof(double) * wpb + 2 * NMAX * sizeof(double) +
                        (size_t(ntiles) * 16 + NMAX * (NMAX - 1) / 2 + 1) * sizeof(int);
    auto kfn = gpr_wdmma_kernel<NMAX>;
    VX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    VX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 32 * wpb, smem));
    if (per_sm < 1) per_sm = 1;
    int blocks = (va.num_items + wpb - 1) / wpb;
    const int cap = sm_count() * per_sm;
    if (blocks > cap) blocks = cap;
    kfn<<<blocks, 32 * wpb, smem, s>>>(va, va.M, mm);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

template <bool VOXEL>
static int launch_generic(const VoxelSolveArgs& va, const ProblemArgs& pa, int num_items, int n_max,
                          int m_max, DevBuf& work, cudaStream_t s) {
    if (num_items <= 0) return VX_OK;
    const int64_t per = int64_t(n_max > m_max ? n_max : m_max) * 3 + int64_t(n_max) * 2 +
                        2 * int64_t(n_max) + m_max + int64_t(n_max) * n_max +
                        int64_t(n_max) * (m_max + 1) + 16;
    int blocks = num_items;
    const int cap = sm_count() * 4;
    if (blocks > cap) blocks = cap;
    // bound the workspace to ~4 GiB
    const int64_t max_blocks = (int64_t(4) << 30) / (per * 8);
    if (blocks > max_blocks) blocks = int(max_blocks > 0 ? max_blocks : 1);
    VX_TRY(work.reserve(size_t(per) * blocks * sizeof(double), s));
    GenericWork gw{work.as<double>(), per, n_max, m_max};
    gpr_generic_kernel<VOXEL><<<blocks, GB, 0, s>>>(va, pa, gw);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

int launch_pca_prepass(const VoxelSolveArgs& a, int S, long long* bucket_counts, cudaStream_t s) {
    if (S <= 0) return VX_OK;
    k_pca_prepass<<<(S + 127) / 128, 128, 0, s>>>(a, S, bucket_counts);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

int launch_bucket_items(const VoxelSolveArgs& a, int S, int32_t* items, const long long* base,
                        long long* fill, cudaStream_t s) {
    if (S <= 0) return VX_OK;
    k_bucket_items<<<(S + 255) / 256, 256, 0, s>>>(a.cand_n, a.cand_axis, S, items, base, fill);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

int launch_voxel_solve(const VoxelSolveArgs& a, int max_n, DevBuf& work, cudaStream_t s,
                       int bucket) {
    ProblemArgs none{};
    if (a.num_items <= 0) return VX_OK;
    const int mm = a.n_s * a.n_r;
    if (mm > MAX_MM) {
        set_error("n_s * n_r = %d exceeds %d", mm, MAX_MM);
        return VX_E_INPUT;
    }
    // A/B hook: VX_PANEL_FROM=k routes the tile buckets whose lower bound is >= k
    // (64, 96, 128) to the panel kernel
    if (const char* e = getenv("VX_PANEL_FROM")) {
        const int from = atoi(e);
        const int lo = bucket == 6 ? 64 : bucket == 3 ? 96 : bucket == 7 ? 128 : -1;
        if (lo >= 0 && lo >= from) return launch_panel<true>(a, none, a.num_items, max_n, a.M, mm, work, s);
    }
    switch (bucket) {
        case 0: return launch_wdmma<16>(a, mm, s);
        case 1: return launch_wdmma<24>(a, mm, s);
        case 5: return launch_wdmma<32>(a, mm, s);
        case 2:   // 32 < n <= 64
            return launch_tile<8, T64_CFG, true>(a, none, a.num_items, a.M, mm, s);
        case 6:   // 64 < n <= 96
            return launch_tile<T96_NRB, T96_CFG, true>(a, none, a.num_items, a.M, mm, s);
        case 3:   // 96 < n <= 128: two CTAs per SM, one 8-column tile per warp per pass
            return launch_tile<16, T128_CFG, true>(a, none, a.num_items, a.M, mm, s);
        case 7:   // 128 < n <= 160
            // one 12-warp tile CTA per SM (measured: 2.51 -> 2.36 ms vs gpr_big_kernel<12>)
            if (a.M + 1 <= 96)
                return launch_tile<20, 1, T160_NW, 1, T160_ROWS, true>(a, none, a.num_items, a.M, mm, s);
            return launch_cta<true>(a, none, a.num_items, max_n < 160 ? max_n : 160, a.M, mm, work, s);
        default:   // n > 160: augmented panel Cholesky on a team of CTAs
            if (!getenv("VX_OLD_BIG"))
                return launch_panel<true>(a, none, a.num_items, max_n, a.M, mm, work, s);
            if (a.M + 1 <= 96) return launch_big<12, true>(a, none, a.num_items, max_n, a.M, mm, work, s);
            return launch_cta<true>(a, none, a.num_items, max_n, a.M, mm, work, s);
    }
}

int launch_problem_solve(const VxGprBatch& b, const int32_t* d_items, int32_t count, int max_n,
                         int max_m, DevBuf& work, cudaStream_t s, int bucket) {
    VoxelSolveArgs none{};
    ProblemArgs pa{d_items, count, b.d_x_off, b.d_q_off, b.d_x, b.d_f, b.d_noise, b.d_xs,
                   b.d_lam, b.jitter, b.kernel, b.d_mu, b.d_var, b.d_full, b.d_full_off,
                   b.d_status};
    if (count <= 0) return VX_OK;
    if (b.d_full == nullptr) {
        if (bucket == 0) return launch_warp<16, false>(none, pa, count, max_m, 1, s);
        if (bucket == 1) return launch_warp<24, false>(none, pa, count, max_m, 1, s);
        if (bucket == 5) return launch_warp<32, false>(none, pa, count, max_m, 1, s);
        if (bucket == 2) return launch_tile<8, T64_CFG, false>(none, pa, count, max_m, 1, s);
        if (bucket == 6) return launch_tile<T96_NRB, T96_CFG, false>(none, pa, count, max_m, 1, s);
        if (bucket == 3) return launch_tile<16, T128_CFG, false>(none, pa, count, max_m, 1, s);

        if (!getenv("VX_OLD_BIG")) return launch_panel<false>(none, pa, count, max_n, max_m, 1, work, s);
        return launch_big<12, false>(none, pa, count, max_n, max_m, 1, work, s);
    }
    return launch_generic<false>(none, pa, count, max_n, max_m, work, s);
}

}  // namespace vx

#ifdef VX_PHASE_TIMING
// diagnostics-build export: copy out and reset the per-phase cycle sums
extern "C" int vx_phase_cycles(unsigned long long* out, int max_phases) {
    unsigned long long h[20];
    if (cudaMemcpyFromSymbol(h, vx::g_phase_cycles, sizeof(h)) != cudaSuccess) return -1;
    const unsigned long long z[20] = {};
    cudaMemcpyToSymbol(vx::g_phase_cycles, z, sizeof(z));
    const int k = max_phases < 20 ? max_phases : 20;
    for (int i = 0; i < k; ++i) out[i] = h[i];
    return k;
}
#endif

#ifdef VX_PHASE_TIMING
// diagnostics-build microbenchmark: cycles of one diag_block_factor call (one
// warp, 32x32 SPD block in global memory, repeated `iters` times)
namespace vx {
__global__ void k_diag_bench(const double* P, int iters, unsigned long long* out) {
    extern __shared__ __align__(16) double sm[];
    double* LD = sm;
    double* LI = sm + PNB * PLD;
    double* DINV = LI + PNB * PLD;
    const int lane = threadIdx.x & 31;
    bool ok = true;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) ok &= diag_block_factor(P, PNB, LD, LI, DINV, lane);
    const long long t1 = clock64();
    if (lane == 0) out[0] = (unsigned long long)(t1 - t0) / iters + (ok ? 0 : 1ull << 62);
}
}  // namespace vx
extern "C" int vx_diag_parts(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, vx::g_diag_t, 8 * sizeof(unsigned long long));
    const unsigned long long z[8] = {};
    cudaMemcpyToSymbol(vx::g_diag_t, z, sizeof(z));
    return 0;
}
extern "C" int vx_diag_bench(int iters, unsigned long long* cycles) {
    double h[32 * 32];
    for (int c = 0; c < 32; ++c)
        for (int r = 0; r < 32; ++r) h[c * 32 + r] = (r == c ? 40.0 : 1.0 / (1.0 + r + c));
    double* d = nullptr;
    unsigned long long* o = nullptr;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 8);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    vx::k_diag_bench<<<1, 32, (2 * 32 * vx::PLD + 32) * 8>>>(d, iters, o);
    cudaMemcpy(cycles, o, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(o);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
#endif
