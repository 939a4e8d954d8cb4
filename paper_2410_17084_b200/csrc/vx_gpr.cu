// Batched per-voxel Gaussian-process regression, FP64, sm_100a.
//
// Replaces gpr.py:57-311 (select_value_axis, make_mesh_grid, kernel_matrix,
// gpr_solve, densify_frame's per-voxel body) and voxel_map.py:242-261 /
// 344-355 (apply_prediction's fold-back and reclassification).
//
// Two kernel families, chosen per training-set size n (size buckets):
//
//  * team kernel (n <= 64): a "team" of 32*ceil((m+1)/32) threads owns one
//    voxel at a time; several teams per CTA, each synchronised by its own
//    named barrier.  The team builds A = K + diag(noise) in shared memory,
//    factorises it (one warp, rows in registers, warp shuffles, for n <= 32;
//    team-parallel left-looking in shared memory for n <= 64), then every
//    thread owns one right-hand side column of [f | K*] and runs a
//    left-looking forward substitution with the column held in registers:
//        w = L^-1 k*_c,  sigma^2_c = 1 - |w|^2,  mu_c = w . (L^-1 f).
//    K* is never materialised: for the SE kernel on the voxel's regular grid
//    k*(x_i, g) = exp(-lam dx^2) exp(-lam dy^2) is separable, so the team
//    tabulates 2 * n * (n_s n_r) exponentials instead of n * (n_s n_r)^2.
//  * generic kernel (any n): one CTA per voxel, A/L (column-major) and W in a
//    per-CTA global workspace (L2-resident), left-looking Cholesky and a
//    row-blocked forward substitution.  Serves the Livox-style tail and
//    re-fits whose raw ∪ pseudo training sets grow past 64 points.
//
// Both write the prediction (points, colours, clipped variances) into the
// voxel's prediction slot — which is also the pseudo-observation set of its
// next solve — and update the lifecycle state in the same kernel.
#include <cfloat>
#include <cmath>

#include "vx_common.cuh"
#include "vx_internal.h"

namespace vx {

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
// shared-memory carve-up of one team (small kernel)
// ---------------------------------------------------------------------------
template <int NMAX>
struct TeamLayout {
    static constexpr int LD = NMAX + 1;           // odd stride: conflict-free rows
    int mmax;                                     // max query count
    __host__ __device__ static int doubles(int mmax) {
        return NMAX * 2 /*X*/ + NMAX /*F*/ + NMAX /*NZ*/ + NMAX /*Z*/ +
               NMAX * LD /*L (also 3-D staging)*/ + 2 * NMAX * MAX_MM /*EA,EB*/ +
               mmax /*VAR*/ + 8 /*misc*/;
    }
};

struct TeamPtrs {
    double *X, *F, *NZ, *Z, *L, *EA, *EB, *VAR, *misc;
};

template <int NMAX>
__device__ __forceinline__ TeamPtrs carve(double* base, int mmax) {
    TeamPtrs p;
    p.X = base;
    p.F = p.X + NMAX * 2;
    p.NZ = p.F + NMAX;
    p.Z = p.NZ + NMAX;
    p.L = p.Z + NMAX;
    p.EA = p.L + NMAX * TeamLayout<NMAX>::LD;
    p.EB = p.EA + NMAX * MAX_MM;
    p.VAR = p.EB + NMAX * MAX_MM;
    p.misc = p.VAR + mmax;
    return p;
}

// triangular index -> (i, j), j <= i
__device__ __forceinline__ void tri_decode(int idx, int* i, int* j) {
    int r = int((sqrt(8.0 * idx + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= idx) ++r;
    while (r * (r + 1) / 2 > idx) --r;
    *i = r;
    *j = idx - r * (r + 1) / 2;
}

// build A = K + diag(noise) (+ jitter on the retry) into row-major L
template <int LD>
__device__ void team_build_A(const TeamPtrs& t, int n, double lam, int kind, double jit,
                             int tid, int TS) {
    const int tot = n * (n + 1) / 2;
    for (int idx = tid; idx < tot; idx += TS) {
        int i, j;
        tri_decode(idx, &i, &j);
        double v;
        if (i == j) {
            // K_ii = exp(-lam * 0) = 1 exactly, then + noise (gpr.py:185),
            // then + jitter on the retry (gpr.py:189)
            v = xadd(1.0, t.NZ[i]);
            if (jit != 0.0) v = xadd(v, jit);
        } else {
            double d2 = dist2_exact(t.X[2 * i], t.X[2 * i + 1], t.X[2 * j], t.X[2 * j + 1]);
            v = kernel_value(kind, lam, d2);
        }
        t.L[i * LD + j] = v;
    }
}

// Cholesky of the n x n (n <= 32) lower triangle in t.L by one warp; row i in
// lane i's registers.  Fails (returns false) on a pivot that is not > 0,
// which is dpotrf's rule (pivot <= 0 or NaN).
template <int LD>
__device__ bool warp_cholesky32(double* L, int n, int lane) {
    double a[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = (lane < n && j <= lane) ? L[lane * LD + j] : 0.0;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if (k < n && ok) {
            double akk = __shfl_sync(FULL, a[k], k);
            if (!(akk > 0.0)) {
                ok = false;
            } else {
                double lkk = sqrt(akk);
                if (lane == k) a[k] = lkk;
                else if (lane > k) a[k] = a[k] / lkk;
                double lik = a[k];
#pragma unroll
                for (int j = k + 1; j < 32; ++j) {
                    if (j < n) {
                        double ljk = __shfl_sync(FULL, a[k], j);
                        if (lane >= j) a[j] = fma(-lik, ljk, a[j]);
                    }
                }
            }
        }
    }
    if (ok && lane < n) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j <= lane) L[lane * LD + j] = a[j];
    }
    __syncwarp();
    return ok;
}

// team-parallel left-looking Cholesky in shared memory (row-major, odd LD):
// column j: s_i = A_ij - sum_{k<j} L_ik L_jk for i >= j; L_jj = sqrt(s_j);
// L_ij = s_i / L_jj.  Returns false on a non-positive pivot (uniform).
template <int LD>
__device__ bool team_cholesky(double* L, int n, int tid, int TS, int bar, double* flag) {
    for (int j = 0; j < n; ++j) {
        for (int i = j + tid; i < n; i += TS) {
            const double* Li = L + i * LD;
            const double* Lj = L + j * LD;
            double s0 = Li[j], s1 = 0.0;
            int k = 0;
            for (; k + 1 < j; k += 2) {
                s0 = fma(-Li[k], Lj[k], s0);
                s1 = fma(-Li[k + 1], Lj[k + 1], s1);
            }
            if (k < j) s0 = fma(-Li[k], Lj[k], s0);
            L[i * LD + j] = s0 + s1;
        }
        team_sync(bar, TS);
        double d = L[j * LD + j];
        if (!(d > 0.0)) return false;
        double ljj = sqrt(d);
        for (int i = j + 1 + tid; i < n; i += TS) L[i * LD + j] = L[i * LD + j] / ljj;
        team_sync(bar, TS);
        if (tid == 0) L[j * LD + j] = ljj;
        // the diagonal write is read only after the next barrier
    }
    team_sync(bar, TS);
    return true;
}

// ---------------------------------------------------------------------------
// the team kernel
// ---------------------------------------------------------------------------
template <int NMAX>
struct TeamBounds {
    static constexpr int MAXT = NMAX <= 32 ? 384 : 256;
};

template <int NMAX, bool VOXEL>
__global__ void __launch_bounds__(TeamBounds<NMAX>::MAXT) gpr_team_kernel(VoxelSolveArgs va, ProblemArgs pa,
                                                       int TS, int teams, int mmax) {
    extern __shared__ double smem[];
    constexpr int LD = TeamLayout<NMAX>::LD;
    const int team = threadIdx.x / TS;
    const int tid = threadIdx.x % TS;
    const int bar = 1 + team;
    const int lane = threadIdx.x & 31;
    const int twarp = tid >> 5;
    TeamPtrs t = carve<NMAX>(smem + size_t(team) * TeamLayout<NMAX>::doubles(mmax), mmax);
    int* imisc = reinterpret_cast<int*>(t.misc + 4);

    const int num_items = VOXEL ? va.num_items : pa.num_items;
    for (int it = blockIdx.x * teams + team; it < num_items; it += gridDim.x * teams) {
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
            // ---- stage raw ∪ pseudo (voxel_map.py:196-200) as 3-D points in L
            double* P3 = t.L;
            const bool hp = va.has_pred[vid] != 0;
            for (int r = tid; r < n; r += TS) {
                const double* src;
                double nz;
                if (r < cnt) {
                    src = va.raw_xyz + (off + r) * 3;
                    nz = va.sensor_var;
                } else {
                    int64_t pr = int64_t(slot) * m + (r - cnt);
                    src = va.pred_xyz + pr * 3;
                    nz = va.pred_var[pr];
                }
                P3[r * 3 + 0] = src[0];
                P3[r * 3 + 1] = src[1];
                P3[r * 3 + 2] = src[2];
                t.NZ[r] = nz;
            }
            (void)hp;
            team_sync(bar, TS);
            // ---- value axis by PCA (gpr.py:57-78), warp 0 of the team
            if (twarp == 0) {
                double mx = 0.0, my = 0.0, mz = 0.0;
                if (lane == 0) {
                    // pts.mean(axis=0): sequential accumulation, then / n
                    for (int r = 0; r < n; ++r) {
                        mx = xadd(mx, P3[r * 3]);
                        my = xadd(my, P3[r * 3 + 1]);
                        mz = xadd(mz, P3[r * 3 + 2]);
                    }
                    mx = xdiv(mx, double(n));
                    my = xdiv(my, double(n));
                    mz = xdiv(mz, double(n));
                }
                mx = __shfl_sync(FULL, mx, 0);
                my = __shfl_sync(FULL, my, 0);
                mz = __shfl_sync(FULL, mz, 0);
                double c[6] = {0, 0, 0, 0, 0, 0};
                for (int r = lane; r < n; r += 32) {
                    double dx = xsub(P3[r * 3], mx), dy = xsub(P3[r * 3 + 1], my),
                           dz = xsub(P3[r * 3 + 2], mz);
                    c[0] = fma(dx, dx, c[0]);
                    c[1] = fma(dx, dy, c[1]);
                    c[2] = fma(dx, dz, c[2]);
                    c[3] = fma(dy, dy, c[3]);
                    c[4] = fma(dy, dz, c[4]);
                    c[5] = fma(dz, dz, c[5]);
                }
#pragma unroll
                for (int k = 0; k < 6; ++k)
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) c[k] += __shfl_xor_sync(FULL, c[k], o);
                if (lane == 0) {
                    int ax = -1;
                    if (n >= 3) {
                        for (int k = 0; k < 6; ++k) c[k] /= double(n);
                        double ev[3], v0[3];
                        eig3_sym(c, ev, v0, nullptr);
                        if (!(ev[2] <= 1e-18 || ev[1] <= 1e-9 * ev[2])) {
                            double w0 = fabs(v0[0]), w1 = fabs(v0[1]), w2 = fabs(v0[2]);
                            // argmax over (z, y, x): ties prefer z, then y
                            ax = 2;
                            double best = w2;
                            if (w1 > best) { ax = 1; best = w1; }
                            if (w0 > best) { ax = 0; }
                        }
                    }
                    imisc[0] = ax;
                }
            }
            team_sync(bar, TS);
            axis = imisc[0];
            if (axis < 0) {
                if (tid == 0) {
                    va.cand_status[s] = VX_ST_DEGENERATE;
                    uint8_t st = va.state[vid];
                    va.cand_before[s] = st;
                    va.cand_after[s] = st;
                }
                team_sync(bar, TS);
                continue;
            }
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            for (int r = tid; r < n; r += TS) {
                t.X[2 * r] = P3[r * 3 + pa_];
                t.X[2 * r + 1] = P3[r * 3 + pb_];
                t.F[r] = P3[r * 3 + axis];
            }
            team_sync(bar, TS);
            if (tid == 0) {
                const double* F = t.F;
                double sum = np_pairwise_sum([F](int i) { return F[i]; }, n);
                t.misc[0] = xdiv(sum, double(n));     // f.mean() (gpr.py:291)
            }
            team_sync(bar, TS);
            mean_f = t.misc[0];
            for (int r = tid; r < n; r += TS) t.F[r] = xsub(t.F[r], mean_f);
        } else {
            s = pa.items[it];
            xo = pa.x_off[s];
            qo = pa.q_off[s];
            n = int(pa.x_off[s + 1] - xo);
            m = int(pa.q_off[s + 1] - qo);
            lam = pa.lam[s];
            jitter = pa.jitter;
            kind = pa.kernel;
            for (int r = tid; r < n; r += TS) {
                t.X[2 * r] = pa.x[(xo + r) * 2];
                t.X[2 * r + 1] = pa.x[(xo + r) * 2 + 1];
                t.F[r] = pa.f[xo + r];
                t.NZ[r] = pa.noise[xo + r];
            }
        }
        team_sync(bar, TS);

        // ---- A = K + diag(noise); Cholesky; one jitter retry (gpr.py:184-194)
        bool ok = false;
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            team_build_A<LD>(t, n, lam, kind, attempt ? jitter : 0.0, tid, TS);
            team_sync(bar, TS);
            if constexpr (NMAX <= 32) {
                if (twarp == 0) {
                    bool r = warp_cholesky32<LD>(t.L, n, lane);
                    if (lane == 0) imisc[1] = r ? 1 : 0;
                }
                team_sync(bar, TS);
                ok = imisc[1] != 0;
            } else {
                ok = team_cholesky<LD>(t.L, n, tid, TS, bar, t.misc);
            }
            team_sync(bar, TS);
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
            team_sync(bar, TS);
            continue;
        }

        // ---- voxel grid (gpr.py:104-120, 262-266) and separable SE tables
        double lo0 = 0, lo1 = 0, sp0 = 0, sp1 = 0;
        const bool sep = VOXEL && kind == VX_KERNEL_SE;
        if constexpr (VOXEL) {
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            lo0 = xmul(double(va.keys[vid * 3 + pa_]), va.voxel_size);
            lo1 = xmul(double(va.keys[vid * 3 + pb_]), va.voxel_size);
            sp0 = xsub(xadd(lo0, va.voxel_size), lo0);    // hi - lo
            sp1 = xsub(xadd(lo1, va.voxel_size), lo1);
            if (sep) {
                for (int e = tid; e < 2 * n * mm; e += TS) {
                    int which = e / (n * mm);
                    int rem = e - which * n * mm;
                    int i = rem / mm, r = rem - i * mm;
                    double lo = which ? lo1 : lo0, sp = which ? sp1 : sp0;
                    double g = xadd(lo, xdiv(xmul(double(r) + 0.5, sp), double(mm)));
                    double d = xsub(t.X[2 * i + which], g);
                    (which ? t.EB : t.EA)[i * mm + r] = exp(xmul(-lam, xmul(d, d)));
                }
            }
        }
        team_sync(bar, TS);

        // ---- forward substitution: thread owns column c of [f | K*]
        const int ncols = m + 1;
        const int passes = (ncols + TS - 1) / TS;
        for (int pass = 0; pass < passes; ++pass) {
            const int c = pass * TS + tid;
            const bool active = c < ncols;
            const int q = c - 1;
            double g0 = 0, g1 = 0;
            int ri = 0, si = 0;
            if (active && c > 0) {
                if constexpr (VOXEL) {
                    const int nr2 = va.n_r * va.n_r;
                    const int sr = q / (va.n_s * nr2);
                    const int rem = q - sr * va.n_s * nr2;
                    const int sc = rem / nr2;
                    const int rem2 = rem - sc * nr2;
                    const int fr = rem2 / va.n_r, fc = rem2 - fr * va.n_r;
                    ri = sr * va.n_r + fr;
                    si = sc * va.n_r + fc;
                    g0 = xadd(lo0, xdiv(xmul(double(ri) + 0.5, sp0), double(mm)));
                    g1 = xadd(lo1, xdiv(xmul(double(si) + 0.5, sp1), double(mm)));
                } else {
                    g0 = pa.xs[(qo + q) * 2];
                    g1 = pa.xs[(qo + q) * 2 + 1];
                }
            }
            double w[NMAX];
            double ss = 0.0;
#pragma unroll
            for (int i = 0; i < NMAX; ++i) {
                if (i < n) {
                    double rhs;
                    if (c == 0) rhs = t.F[i];
                    else if (!active) rhs = 0.0;
                    else if (sep) rhs = t.EA[i * mm + ri] * t.EB[i * mm + si];
                    else rhs = kernel_value(kind, lam, dist2_exact(t.X[2 * i], t.X[2 * i + 1], g0, g1));
                    const double* Li = t.L + i * LD;
                    double b0 = rhs, b1 = 0.0;
#pragma unroll
                    for (int j = 0; j + 1 < i; j += 2) {
                        b0 = fma(-Li[j], w[j], b0);
                        b1 = fma(-Li[j + 1], w[j + 1], b1);
                    }
                    if (i & 1) b0 = fma(-Li[i - 1], w[i - 1], b0);
                    w[i] = (b0 + b1) / Li[i];
                    ss = fma(w[i], w[i], ss);
                }
            }
            if (c == 0) {
#pragma unroll
                for (int i = 0; i < NMAX; ++i)
                    if (i < n) t.Z[i] = w[i];
            }
            team_sync(bar, TS);
            const bool query = active && c > 0;
            double mu = 0.0, var = 0.0, pos[3] = {0, 0, 0}, colr[3] = {0, 0, 0};
            if (query) {
                double mu0 = 0.0, mu1 = 0.0;
#pragma unroll
                for (int i = 0; i + 1 < NMAX; i += 2) {
                    if (i < n) mu0 = fma(w[i], t.Z[i], mu0);
                    if (i + 1 < n) mu1 = fma(w[i + 1], t.Z[i + 1], mu1);
                }
                mu = mu0 + mu1;
                var = 1.0 - ss;
                if constexpr (VOXEL) {
                    var = var < 0.0 ? 0.0 : var;     // np.clip(., 0, None)
                    t.VAR[q] = var;
                    const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
                    pos[axis] = xadd(mu, mean_f);
                    pos[pa_] = g0;
                    pos[pb_] = g1;
                    // nearest training point in the parameter plane (gpr.py:304-305)
                    double best = INFINITY;
                    int bi = 0;
                    for (int i = 0; i < n; ++i) {
                        double d2 = dist2_exact(g0, g1, t.X[2 * i], t.X[2 * i + 1]);
                        if (d2 < best) { best = d2; bi = i; }
                    }
                    const double* cs = bi < cnt ? va.raw_rgb + (off + bi) * 3
                                                : va.pred_rgb + (int64_t(slot) * m + (bi - cnt)) * 3;
                    colr[0] = cs[0];
                    colr[1] = cs[1];
                    colr[2] = cs[2];
                } else {
                    pa.mu[qo + q] = mu;
                    pa.var[qo + q] = var;
                }
            }
            if constexpr (VOXEL) {
                // every read of the previous prediction precedes any write
                team_sync(bar, TS);
                if (query) {
                    const int64_t pr = int64_t(slot) * m + q;
                    va.pred_xyz[pr * 3 + 0] = pos[0];
                    va.pred_xyz[pr * 3 + 1] = pos[1];
                    va.pred_xyz[pr * 3 + 2] = pos[2];
                    va.pred_rgb[pr * 3 + 0] = colr[0];
                    va.pred_rgb[pr * 3 + 1] = colr[1];
                    va.pred_rgb[pr * 3 + 2] = colr[2];
                    va.pred_var[pr] = var;
                }
            }
            team_sync(bar, TS);
        }
        if (tid == 0) {
            if constexpr (VOXEL) {
                const double* V = t.VAR;
                double mv = xdiv(np_pairwise_sum([V](int i) { return V[i]; }, m), double(m));
                uint8_t before = va.state[vid];
                uint8_t after = mv <= va.eta ? VX_CONVERGED : VX_ACTIVE;
                va.state[vid] = after;
                va.value_axis[vid] = int8_t(axis);
                va.has_pred[vid] = 1;
                va.cand_status[s] = VX_ST_OK;
                va.cand_before[s] = before;
                va.cand_after[s] = after;
            } else {
                pa.status[s] = VX_ST_OK;
            }
        }
        team_sync(bar, TS);
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
    __shared__ double red[32];
    __shared__ int ishared[4];
    __shared__ double dshared[4];
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
            for (int r = tid; r < n; r += GB) {
                const double* src;
                double nz;
                if (r < cnt) {
                    src = va.raw_xyz + (off + r) * 3;
                    nz = va.sensor_var;
                } else {
                    int64_t pr = int64_t(slot) * m + (r - cnt);
                    src = va.pred_xyz + pr * 3;
                    nz = va.pred_var[pr];
                }
                P3[r * 3 + 0] = src[0];
                P3[r * 3 + 1] = src[1];
                P3[r * 3 + 2] = src[2];
                NZ[r] = nz;
            }
            __syncthreads();
            if (tid == 0) {
                double mx = 0, my = 0, mz = 0;
                for (int r = 0; r < n; ++r) {
                    mx = xadd(mx, P3[r * 3]);
                    my = xadd(my, P3[r * 3 + 1]);
                    mz = xadd(mz, P3[r * 3 + 2]);
                }
                dshared[0] = xdiv(mx, double(n));
                dshared[1] = xdiv(my, double(n));
                dshared[2] = xdiv(mz, double(n));
            }
            __syncthreads();
            const double mx = dshared[0], my = dshared[1], mz = dshared[2];
            double c[6] = {0, 0, 0, 0, 0, 0};
            for (int r = tid; r < n; r += GB) {
                double dx = xsub(P3[r * 3], mx), dy = xsub(P3[r * 3 + 1], my),
                       dz = xsub(P3[r * 3 + 2], mz);
                c[0] = fma(dx, dx, c[0]);
                c[1] = fma(dx, dy, c[1]);
                c[2] = fma(dx, dz, c[2]);
                c[3] = fma(dy, dy, c[3]);
                c[4] = fma(dy, dz, c[4]);
                c[5] = fma(dz, dz, c[5]);
            }
            for (int k = 0; k < 6; ++k) c[k] = block_sum(c[k], red);
            if (tid == 0) {
                int ax = -1;
                if (n >= 3) {
                    for (int k = 0; k < 6; ++k) c[k] /= double(n);
                    double ev[3], v0[3];
                    eig3_sym(c, ev, v0, nullptr);
                    if (!(ev[2] <= 1e-18 || ev[1] <= 1e-9 * ev[2])) {
                        double w0 = fabs(v0[0]), w1 = fabs(v0[1]), w2 = fabs(v0[2]);
                        ax = 2;
                        double best = w2;
                        if (w1 > best) { ax = 1; best = w1; }
                        if (w0 > best) { ax = 0; }
                    }
                }
                ishared[0] = ax;
            }
            __syncthreads();
            axis = ishared[0];
            if (axis < 0) {
                if (tid == 0) {
                    va.cand_status[s] = VX_ST_DEGENERATE;
                    uint8_t st = va.state[vid];
                    va.cand_before[s] = st;
                    va.cand_after[s] = st;
                }
                __syncthreads();
                continue;
            }
            const int pa_ = param_axis_a(axis), pb_ = param_axis_b(axis);
            for (int r = tid; r < n; r += GB) {
                X[2 * r] = P3[r * 3 + pa_];
                X[2 * r + 1] = P3[r * 3 + pb_];
                F[r] = P3[r * 3 + axis];
            }
            __syncthreads();
            if (tid == 0) {
                double sum = np_pairwise_sum([F](int i) { return F[i]; }, n);
                dshared[3] = xdiv(sum, double(n));
            }
            __syncthreads();
            mean_f = dshared[3];
            for (int r = tid; r < n; r += GB) F[r] = xsub(F[r], mean_f);
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
// host launchers
// ---------------------------------------------------------------------------
// one pass over the m+1 right-hand sides whenever m < 1024 (voxel mode
// relies on it: every read of the previous prediction precedes every write)
static int team_threads_for(int m) {
    int ts = ((m + 1 + 31) / 32) * 32;
    return ts > 1024 ? 1024 : ts;
}

template <int NMAX, bool VOXEL>
static int launch_team(const VoxelSolveArgs& va, const ProblemArgs& pa, int num_items, int m_max,
                       cudaStream_t s) {
    const int TS = team_threads_for(m_max);
    int teams = 384 / TS;
    if (teams < 1) teams = 1;
    if (teams > 8) teams = 8;
    if (teams * TS > TeamBounds<NMAX>::MAXT) teams = TeamBounds<NMAX>::MAXT / TS;
    const size_t per_team = size_t(TeamLayout<NMAX>::doubles(m_max)) * sizeof(double);
    const size_t smem_cap = 227 * 1024;
    if (size_t(teams) * per_team > smem_cap) teams = int(smem_cap / per_team);
    if (teams < 1) {
        set_error("team of %d threads exceeds the NMAX=%d kernel bound", TS, NMAX);
        return VX_E_INPUT;
    }
    const size_t smem = size_t(teams) * TeamLayout<NMAX>::doubles(m_max) * sizeof(double);
    auto kfn = gpr_team_kernel<NMAX, VOXEL>;
    VX_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int blocks = (num_items + teams - 1) / teams;
    const int cap = sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) return VX_OK;
    kfn<<<blocks, teams * TS, smem, s>>>(va, pa, TS, teams, m_max);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

template <bool VOXEL>
static int launch_generic(const VoxelSolveArgs& va, const ProblemArgs& pa, int num_items, int n_max,
                          int m_max, DevBuf& work, cudaStream_t s) {
    if (num_items <= 0) return VX_OK;
    const int64_t per = int64_t(n_max > m_max ? n_max : m_max) * 3 + int64_t(n_max) * 2 + 2 * int64_t(n_max) + m_max +
                        int64_t(n_max) * n_max + int64_t(n_max) * (m_max + 1) + 16;
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

int launch_voxel_solve(const VoxelSolveArgs& a, int max_n, DevBuf& work, cudaStream_t s,
                       int bucket) {
    ProblemArgs none{};
    if (a.num_items <= 0) return VX_OK;
    if (a.n_s * a.n_r > MAX_MM) {
        set_error("n_s * n_r = %d exceeds %d", a.n_s * a.n_r, MAX_MM);
        return VX_E_INPUT;
    }
    if (bucket == 0) return launch_team<32, true>(a, none, a.num_items, a.M, s);
    if (bucket == 1 && team_threads_for(a.M) <= TeamBounds<64>::MAXT)
        return launch_team<64, true>(a, none, a.num_items, a.M, s);
    return launch_generic<true>(a, none, a.num_items, max_n, a.M, work, s);
}

int launch_problem_solve(const VxGprBatch& b, const int32_t* d_items, int32_t count, int max_n,
                         int max_m, DevBuf& work, cudaStream_t s, int bucket) {
    VoxelSolveArgs none{};
    ProblemArgs pa{d_items, count, b.d_x_off, b.d_q_off, b.d_x, b.d_f, b.d_noise, b.d_xs,
                   b.d_lam, b.jitter, b.kernel, b.d_mu, b.d_var, b.d_full, b.d_full_off,
                   b.d_status};
    if (count <= 0) return VX_OK;
    if (b.d_full == nullptr && team_threads_for(max_m) <= TeamBounds<32>::MAXT) {
        if (bucket == 0) return launch_team<32, false>(none, pa, count, max_m, s);
        if (bucket == 1 && team_threads_for(max_m) <= TeamBounds<64>::MAXT)
            return launch_team<64, false>(none, pa, count, max_m, s);
    }
    return launch_generic<false>(none, pa, count, max_n, max_m, work, s);
}

}  // namespace vx
