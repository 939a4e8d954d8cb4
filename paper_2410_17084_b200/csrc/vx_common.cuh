// Shared device helpers for the voxel-GPR hot path (sm_100a only).
//
// Everything numeric here is FP64: SURVEY.md §0-5 measured that every FP32
// variant of the per-voxel GPR misses the reference's 1e-9 relative parity by
// 20-700x, so the roofline of the solve kernels is the FP64 FMA pipe.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/voxgpr.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "voxgpr is written for sm_100a (B200) only"
#endif

namespace vx {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint64_t EMPTY_KEY = ~0ull;
constexpr int KEY_BITS = 21;                        // per axis, offset binary
constexpr int64_t KEY_BIAS = int64_t(1) << (KEY_BITS - 1);   // 2^20
constexpr int64_t KEY_LIM = KEY_BIAS;               // |k| < 2^20 representable

// ---------------------------------------------------------------------------
// exact IEEE helpers: the reference's NumPy expressions are evaluated
// operation by operation without FMA contraction; where bit-exactness is a
// parity gate (grid coordinates, nearest-colour distances, keys) we use the
// _rn intrinsics so nvcc cannot contract them.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }

// squared distance in the parameter plane, NumPy order ((dx**2) + (dy**2))
// (gpr.py:129 and gpr.py:304)
__device__ __forceinline__ double dist2_exact(double ax, double ay, double bx, double by) {
    double dx = xsub(ax, bx), dy = xsub(ay, by);
    return xadd(xmul(dx, dx), xmul(dy, dy));
}

// ---------------------------------------------------------------------------
// keys: pack a lattice triple into 63 bits (21 bits per axis, offset binary)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t pack_key(int64_t a, int64_t b, int64_t c) {
    return (uint64_t(a + KEY_BIAS) << (2 * KEY_BITS)) | (uint64_t(b + KEY_BIAS) << KEY_BITS) |
           uint64_t(c + KEY_BIAS);
}
__host__ __device__ __forceinline__ void unpack_key(uint64_t k, int64_t* a, int64_t* b, int64_t* c) {
    const uint64_t m = (uint64_t(1) << KEY_BITS) - 1;
    *a = int64_t((k >> (2 * KEY_BITS)) & m) - KEY_BIAS;
    *b = int64_t((k >> KEY_BITS) & m) - KEY_BIAS;
    *c = int64_t(k & m) - KEY_BIAS;
}
// murmur3 finaliser: spreads spatially adjacent keys over the table and over
// shards (voxel owner = mix(key) mod world)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

// ---------------------------------------------------------------------------
// NumPy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum): n < 8 sequential; n <= 128 eight strided accumulators
// combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail;
// larger n splits at n/2 rounded down to a multiple of 8.  Used for the
// reductions the reference evaluates with ndarray.sum()/mean() on contiguous
// 1-D data (f.mean() gpr.py:291, variances.mean() voxel_map.py:170, subgrid
// weight sums splat_init.py:94), so those are bit-exact.
// `get(i)` returns element i.
// ---------------------------------------------------------------------------
template <typename Get>
__device__ double np_pairwise_block(Get get, int lo, int n) {
    if (n < 8) {
        double s = -0.0;          // NumPy starts the plain loop from -0.0
        for (int i = 0; i < n; ++i) s = xadd(s, get(lo + i));
        return s;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = get(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = xadd(r[j], get(lo + i + j));
    }
    double res = xadd(xadd(xadd(r[0], r[1]), xadd(r[2], r[3])),
                      xadd(xadd(r[4], r[5]), xadd(r[6], r[7])));
    for (; i < n; ++i) res = xadd(res, get(lo + i));
    return res;
}

// Warp-cooperative np_pairwise_sum of a shared-memory array: the eight strided
// accumulators live in lanes 0-7 and are combined with shuffles in NumPy's
// order, so the result is bit-identical to np_pairwise_block.  All lanes of
// the warp must call it; every lane gets the result.
__device__ __forceinline__ double warp_pairwise_block(const double* a, int n) {
    if (n < 8) {
        double s = -0.0;
        for (int i = 0; i < n; ++i) s = xadd(s, a[i]);
        return s;
    }
    const int lane = threadIdx.x & 31;
    const int full = n - (n % 8);
    double r = 0.0;
    if (lane < 8) {
        r = a[lane];
        for (int i = 8 + lane; i < full; i += 8) r = xadd(r, a[i]);
    }
    r = xadd(r, __shfl_down_sync(FULL, r, 1));   // r0+r1, r2+r3, ...
    r = xadd(r, __shfl_down_sync(FULL, r, 2));   // (r0+r1)+(r2+r3), ...
    r = xadd(r, __shfl_down_sync(FULL, r, 4));
    double res = __shfl_sync(FULL, r, 0);
    for (int i = full; i < n; ++i) res = xadd(res, a[i]);
    return res;
}

template <typename Get>
__device__ double np_pairwise_sum(Get get, int n) {
    // iterative form of the recursive split for n > 128 (depth <= 24)
    if (n <= 128) return np_pairwise_block(get, 0, n);
    int lo_s[32], n_s[32], state[32];
    double acc[32];
    int sp = 0;
    lo_s[0] = 0; n_s[0] = n; state[0] = 0;
    double ret = 0.0;
    while (sp >= 0) {
        int lo = lo_s[sp], cnt = n_s[sp];
        if (cnt <= 128) {
            ret = np_pairwise_block(get, lo, cnt);
            --sp;
            // feed result to parent
            while (sp >= 0) {
                if (state[sp] == 1) {          // left done, start right
                    acc[sp] = ret;
                    state[sp] = 2;
                    int n2 = n_s[sp] / 2;
                    n2 -= n2 % 8;
                    ++sp;
                    lo_s[sp] = lo_s[sp - 1] + n2;
                    n_s[sp] = n_s[sp - 1] - n2;
                    state[sp] = 0;
                    break;
                } else {                       // right done
                    ret = xadd(acc[sp], ret);
                    --sp;
                }
            }
            continue;
        }
        // split: process left half first
        state[sp] = 1;
        int n2 = cnt / 2;
        n2 -= n2 % 8;
        ++sp;
        lo_s[sp] = lo;
        n_s[sp] = n2;
        state[sp] = 0;
    }
    return ret;
}

// np_pairwise_sum of a shared-memory array by a whole warp (n <= 256: at most
// one split level, as for n* <= 256); larger n falls back to the scalar form.
__device__ __forceinline__ double warp_pairwise_sum(const double* a, int n) {
    if (n <= 128) return warp_pairwise_block(a, n);
    if (n <= 256) {
        int n2 = n / 2;
        n2 -= n2 % 8;
        const double left = warp_pairwise_block(a, n2);
        return xadd(left, warp_pairwise_block(a + n2, n - n2));
    }
    return np_pairwise_sum([a](int i) { return a[i]; }, n);
}

// ---------------------------------------------------------------------------
// Symmetric 3x3 eigensolver (cyclic Jacobi, FP64).  Returns eigenvalues in
// ascending order and the eigenvector of the smallest one.  Jacobi is
// accurate to O(eps*|A|/gap) in the eigenvectors — the same accuracy class as
// LAPACK dsyevd used by the reference (numpy.linalg.eigh, gpr.py:72) — which
// keeps the discrete value-axis choice stable on near-isotropic voxels.
// ---------------------------------------------------------------------------
__device__ inline void eig3_sym(const double c[6],  // xx, xy, xz, yy, yz, zz
                                double evals[3], double vmin[3], double V[9]) {
    double a[3][3] = {{c[0], c[1], c[2]}, {c[1], c[3], c[4]}, {c[2], c[4], c[5]}};
    double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (int sweep = 0; sweep < 12; ++sweep) {
        double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
        if (off == 0.0) break;
        const int P[3] = {0, 0, 1}, Q[3] = {1, 2, 2};
        for (int r = 0; r < 3; ++r) {
            int p = P[r], q = Q[r];
            double apq = a[p][q];
            if (apq == 0.0) continue;
            double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
            double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            if (isinf(theta)) t = 0.5 / theta;
            double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
            for (int k = 0; k < 3; ++k) {          // A <- A J
                double akp = a[k][p], akq = a[k][q];
                a[k][p] = cs * akp - sn * akq;
                a[k][q] = sn * akp + cs * akq;
            }
            for (int k = 0; k < 3; ++k) {          // A <- J^T A
                double apk = a[p][k], aqk = a[q][k];
                a[p][k] = cs * apk - sn * aqk;
                a[q][k] = sn * apk + cs * aqk;
            }
            a[p][q] = a[q][p] = 0.0;
            for (int k = 0; k < 3; ++k) {          // V <- V J
                double vkp = v[k][p], vkq = v[k][q];
                v[k][p] = cs * vkp - sn * vkq;
                v[k][q] = sn * vkp + cs * vkq;
            }
        }
    }
    int idx[3] = {0, 1, 2};
    double d[3] = {a[0][0], a[1][1], a[2][2]};
    // sort ascending (3 elements)
    if (d[idx[1]] < d[idx[0]]) { int t = idx[0]; idx[0] = idx[1]; idx[1] = t; }
    if (d[idx[2]] < d[idx[1]]) { int t = idx[1]; idx[1] = idx[2]; idx[2] = t; }
    if (d[idx[1]] < d[idx[0]]) { int t = idx[0]; idx[0] = idx[1]; idx[1] = t; }
    for (int k = 0; k < 3; ++k) evals[k] = d[idx[k]];
    for (int k = 0; k < 3; ++k) vmin[k] = v[k][idx[0]];
    if (V) {
        for (int col = 0; col < 3; ++col)
            for (int k = 0; k < 3; ++k) V[k * 3 + col] = v[k][idx[col]];
    }
}

// select_value_axis (gpr.py:57-78) of n points given by `pt(r)` (a pointer to
// xyz): centred covariance / n, smallest eigenvector, the degeneracy test of
// gpr.py:73-74 and the argmax with ties preferring z, then y (gpr.py:75-77).
// Returns -1 for a degenerate set.  THE one routine both device routes use
// (vx_select_axis_batch and the densify PCA prepass), so they cannot
// disagree: means by sequential accumulation (NumPy reduces axis 0 row by
// row), covariance entries by sequential FMA accumulation.
template <typename PointFn>
__device__ __forceinline__ int pca_value_axis(PointFn pt, int n) {
    if (n < 3) return -1;
    double mx = 0.0, my = 0.0, mz = 0.0;
    for (int r = 0; r < n; ++r) {
        const double* p = pt(r);
        mx = xadd(mx, p[0]);
        my = xadd(my, p[1]);
        mz = xadd(mz, p[2]);
    }
    mx = xdiv(mx, double(n));
    my = xdiv(my, double(n));
    mz = xdiv(mz, double(n));
    double c[6] = {0, 0, 0, 0, 0, 0};
    for (int r = 0; r < n; ++r) {
        const double* p = pt(r);
        const double dx = xsub(p[0], mx), dy = xsub(p[1], my), dz = xsub(p[2], mz);
        c[0] = fma(dx, dx, c[0]);
        c[1] = fma(dx, dy, c[1]);
        c[2] = fma(dx, dz, c[2]);
        c[3] = fma(dy, dy, c[3]);
        c[4] = fma(dy, dz, c[4]);
        c[5] = fma(dz, dz, c[5]);
    }
    for (int k = 0; k < 6; ++k) c[k] = xdiv(c[k], double(n));
    double ev[3], v0[3];
    eig3_sym(c, ev, v0, nullptr);
    if (ev[2] <= 1e-18 || ev[1] <= 1e-9 * ev[2]) return -1;
    const double w0 = fabs(v0[0]), w1 = fabs(v0[1]), w2 = fabs(v0[2]);
    int ax = 2;
    double best = w2;
    if (w1 > best) { ax = 1; best = w1; }
    if (w0 > best) ax = 0;
    return ax;
}

// value axis -> ordered pair of parameter axes (gpr.py:36)
__host__ __device__ __forceinline__ int param_axis_a(int ax) { return ax == 0 ? 1 : (ax == 1 ? 2 : 0); }
__host__ __device__ __forceinline__ int param_axis_b(int ax) { return ax == 0 ? 2 : (ax == 1 ? 0 : 1); }

// Kernel functions with k(q,q)=1.  SE is the reference kernel (gpr.py:123-130):
// exp(-lam * d2) with d2 from dist2_exact.  Matern-3/2 and -5/2 are north-star
// extensions (no reference oracle).
__device__ __forceinline__ double kernel_value(int kind, double lam, double d2) {
    if (kind == VX_KERNEL_SE) return exp(xmul(-lam, d2));
    double r = sqrt(lam * d2);
    if (kind == VX_KERNEL_MATERN32) {
        double s = 1.7320508075688772 * r;
        return (1.0 + s) * exp(-s);
    }
    double s = 2.23606797749979 * r;
    return (1.0 + s + s * s / 3.0) * exp(-s);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp-aggregated counters: lanes hitting the same counter share one atomic
// (the densify bookkeeping kernels otherwise serialise ~1M same-address atomics).
__device__ __forceinline__ unsigned long long agg_add(unsigned long long* ctr, int key,
                                                      unsigned long long v = 1) {
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, key);
    const int leader = __ffs(peers) - 1;
    const int lane = threadIdx.x & 31;
    // every lane adds v, so the warp total for this key is v * popc(peers)
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(ctr + key, v * (unsigned long long)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    return base + v * (unsigned long long)__popc(peers & lt);
}

__device__ __forceinline__ void agg_max(unsigned long long* ctr, unsigned v) {
    const unsigned act = __activemask();
    const unsigned mx = __reduce_max_sync(act, v);
    if ((threadIdx.x & 31) == __ffs(act) - 1) atomicMax(ctr, (unsigned long long)mx);
}

// named barrier for a team of `nthreads` threads (multiple of 32).  The
// non-.aligned form: callers keep every barrier on a team-uniform path, but
// bar.sync (== barrier.sync.aligned) would make any divergence undefined.
__device__ __forceinline__ void team_sync(int id, int nthreads) {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace vx
