// Large-n GPR solve (n > 160): augmented left-looking panel Cholesky on a
// team of CTAs (a thread-block cluster).  Included by vx_gpr.cu (uses its
// staging / epilogue helpers).
//
// gpr_solve (gpr.py:173-205) needs A^-1 applied to the m + 1 right-hand sides
// [f | K*].  Instead of factoring A and then substituting, the kernel factors
// the AUGMENTED matrix
//
//         [ A    ]        rows 0 .. n32-1        A = K + diag(noise), identity-padded to n32
//     M = [      ]
//         [ B^T  ]        rows n32 .. n32+A32-1  B = [f | K*] (zero padded)
//
// column panel by column panel (NB = 32 columns, left-looking):
//
//     P  = M[j:, j:j+32] - L[j:, 0:j] L[j:j+32, 0:j]^T      (phase A, DMMA GEMM)
//     L_dd = chol(P[0:32]) ; L[j+32:, j:j+32] = P[32:] L_dd^-T   (phase B)
//
// so the rows below A come out as W^T = (L^-1 B)^T and the forward
// substitution is part of the factorisation (same flop count, n^3/3 + n^2 m).
// Then mu_q = w_{q+1} . w_0 and sigma^2_q = 1 - |w_{q+1}|^2.  M is generated
// on the fly from the staged training set (the reference formulas:
// exp(-lam d2) with d2 from dist2_exact, diagonal 1 + noise (+ jitter on the
// retry), gpr.py:123-130,184-194).
//
// L lives in a per-team global workspace, panel by panel (panel p holds rows
// [32p, R) of its 32 columns, column-major, ld = R - 32p): 2.7 MB at n = 742,
// L2-resident for the teams in flight.  The GEMM of phase A and the
// triangular update of phase B are split over all warps of the team in 16x32
// row tiles (two CTAs per SM); the 32x32 diagonal block is factored redundantly by one warp of
// every CTA (row per lane in shared memory, left-looking, failure rule of
// dpotrf: a pivot that is not > 0 fails), so the only cross-CTA synchronisation is two cluster
// barriers per panel.  A team takes voxels from the launch's atomic queue
// (largest first, the items are sorted by n before the launch).

// (included inside namespace vx)

constexpr int PNB = 32;          // panel width
constexpr int PW = 8;            // warps per CTA
constexpr int PNT = PW * 32;
constexpr int PLD = 36;          // row stride of L_dd^-1 in shared memory (B fragments: 4 mod 16)
constexpr int PLDL = 33;         // row stride of L_dd (row-per-lane reads: odd)
constexpr int PRT = 16;          // rows per warp tile

struct PanelArgs {
    double* work;                // per-team workspaces
    int64_t per_team;            // doubles per team workspace
    int* queue;                  // launch's item counter
    int* slots;                  // per-team current item
    double* partial;             // per-team epilogue partial sums (C*PW*2*A32 doubles)
    int64_t partial_per_team;
    int csize;                   // CTAs per team (cluster size)
    int nmax, mmax, mm;
};

__host__ __device__ inline int round_up(int v, int r) { return (v + r - 1) / r * r; }
__host__ __device__ inline int64_t panel_base(int R, int p) {
    // sum_{q < p} PNB (R - PNB q)
    return int64_t(PNB) * (int64_t(p) * R - int64_t(PNB) * p * (p - 1) / 2);
}

struct PanelLayout {
    int X, F, NZ, GC, QT, LD, LI, BS, DINV, MU, VAR, COL, FLAG, total;
    __host__ __device__ PanelLayout(int np32, int mcols, int mmax) {
        int o = 0;
        X = o; o += 2 * np32;
        F = o; o += np32;
        NZ = o; o += np32;
        GC = o; o += 2 * MAX_MM;
        QT = o; o += mcols / 2 + 1;       // int32 (ri | si << 16) per column
        LD = o; o += PNB * PLD;           // factored diagonal block (row-major)
        LI = o; o += PNB * PLD;           // its inverse (row-major)
        o = (o + 1) & ~1;                 // 16-byte aligned for cp.async
        BS = o; o += 2 * PNB * PLD;       // phase-A B operand blocks (double buffer)
        DINV = o; o += PNB;               // 1 / L_dd(r, r)
        MU = o; o += mcols;
        VAR = o; o += mcols;
        COL = o; o += 3 * mmax + 1;
        FLAG = o; o += 2;
        total = (o + 1) & ~1;
    }
};

__device__ __forceinline__ void team_sync(int csize) {
    if (csize > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n"
                     "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
        __syncthreads();
    }
}

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// Cholesky factor L_dd and its inverse of the 32x32 diagonal block of a panel,
// by one warp (every CTA of the team runs it redundantly on the same data, so
// all take the same pivot decision).  In: the block P at panel storage `P`
// (column-major, ld `ldp`, lower part used).  Out: LD = L_dd (row-major,
// stride PLDL, lower), LI = L_dd^-1 (row-major, stride PLD, zeros above the
// diagonal; only its four 8x8 diagonal blocks are formed), DINV[r] =
// 1 / L_dd(r, r); returns false when a pivot is not > 0
// (dpotrf's failure rule, gpr.py:187-192).
//
// Left-looking by 8-column blocks, lane = row: the block loads with one
// asynchronous copy wave; per block column the rows at or below it apply the
// finished columns (8 independent FMA chains per lane, the finished rows read
// as shared-memory broadcasts), every lane factors the 8x8 diagonal block in
// its own registers (dpotf2 order: pivot p, scale by 1/sqrt(p), rank-1 update;
// the reciprocal square root is the only transcendental, there is no
// division) and the rows below solve against it in registers.  Then the
// inverses of the four 8x8 diagonal blocks (lane = (block, column)), which
// phase B applies blockwise.
#ifdef VX_PHASE_TIMING
__device__ unsigned long long g_diag_t[8];
#define DIAG_T(i) do { if (lane == 0) { g_diag_t[i] += clock64() - t_; t_ = clock64(); } } while (0)
#else
#define DIAG_T(i) do { } while (0)
#endif
__device__ __noinline__ bool diag_block_factor(const double* __restrict__ P, int ldp, double* LD,
                                               double* LI, double* DINV, int lane) {
#ifdef VX_PHASE_TIMING
    long long t_ = clock64();
#endif
    // P -> LD (row-major, stride PLDL): 32 asynchronous 8-byte copies per lane,
    // one wait (one L2 round trip instead of one per load batch)
    {
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(LD + lane * PLDL));
#pragma unroll
        for (int c = 0; c < PNB; ++c)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d + 8u * c),
                         "l"(P + int64_t(c) * ldp + lane) : "memory");
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
    }
    DIAG_T(0);
    bool good = true;
    // Left-looking by 8-column blocks: lane = row.  (1) rows >= b0 apply every
    // finished block column to their block-column-kb entries (8 independent
    // accumulators per lane, the finished rows read as broadcasts); (2) every
    // lane factors the 8x8 diagonal block in registers; (3) the rows below
    // solve against it in registers.
#pragma unroll 1
    for (int kb = 0; kb < 4; ++kb) {
        const int b0 = 8 * kb;
        double v[8];
        const bool mine = lane >= b0;
        double* row = LD + lane * PLDL;
        if (mine) {
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = row[b0 + c];
#pragma unroll 4
            for (int i = 0; i < b0; ++i) {
                const double li = row[i];
#pragma unroll
                for (int c = 0; c < 8; ++c) v[c] = fma(-li, LD[(b0 + c) * PLDL + i], v[c]);
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) row[b0 + c] = v[c];
        }
        __syncwarp();
        DIAG_T(1);
        double a[36];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c <= r; ++c) a[r * (r + 1) / 2 + c] = LD[(b0 + r) * PLDL + b0 + c];
        double inv[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const double piv = a[c * (c + 1) / 2 + c];
            if (!(piv > 0.0)) good = false;
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
        __syncwarp();
        DIAG_T(2);
        // every row at or below the block solves its 8 entries against the factor:
        // for the block's own rows this reproduces the factorisation operation for
        // operation (the same FMAs in the same order; the diagonal comes out as
        // piv * 1/sqrt(piv)), so no lane has to publish from the replicated a[]
        if (mine) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                v[c] *= inv[c];
#pragma unroll
                for (int k = c + 1; k < 8; ++k) v[k] = fma(-v[c], a[k * (k + 1) / 2 + c], v[k]);
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) row[b0 + c] = v[c];
        }
        double di = 0.0;
#pragma unroll
        for (int r = 0; r < 8; ++r) di = lane == b0 + r ? inv[r] : di;
        if (lane >= b0 && lane < b0 + 8) DINV[lane] = di;
        __syncwarp();
        DIAG_T(3);
    }
    // ---- L^-1: diagonal blocks, lane = (block bl, column c)
    {
        const int bl = lane >> 3, c = lane & 7, b0 = 8 * bl;
        double x[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            double acc = (r == c) ? 1.0 : 0.0;
#pragma unroll
            for (int k = 0; k < r; ++k) acc = fma(-LD[(b0 + r) * PLDL + b0 + k], x[k], acc);
            x[r] = (r < c) ? 0.0 : acc * DINV[b0 + r];
        }
#pragma unroll 4
        for (int r = 0; r < PNB; ++r) LI[r * PLD + lane] = 0.0;        // column `lane`
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 8; ++r) LI[(b0 + r) * PLD + b0 + c] = x[r];
        __syncwarp();
    }
    DIAG_T(4);
    // (the off-diagonal blocks of L_dd^-1 are not needed: phase B solves blockwise)
    DIAG_T(5);
    return good;
}

template <bool VOXEL>
__global__ void __launch_bounds__(PNT, 2) gpr_panel_kernel(VoxelSolveArgs va, ProblemArgs pa,
                                                           PanelArgs pk) {
    extern __shared__ __align__(16) double smem[];
    const int C = pk.csize;
    const int crank = C > 1 ? int(cluster_rank()) : 0;
    const int team = blockIdx.x / C;
    const int nteams = gridDim.x / C;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tig = lane & 3;
    const int NP = round_up(pk.nmax, PNB);
    const int MC = pk.mmax + 1 > 96 ? round_up(pk.mmax + 1, 32) : 96;
    const PanelLayout lay(NP, MC, pk.mmax);
    double* X = smem + lay.X;
    double* F = smem + lay.F;
    double* NZ = smem + lay.NZ;
    double* GC = smem + lay.GC;
    int* QT = reinterpret_cast<int*>(smem + lay.QT);
    double* LD = smem + lay.LD;
    double* LI = smem + lay.LI;
    double* BS = smem + lay.BS;
    double* Lw = pk.work + int64_t(team) * pk.per_team;
    double* part = pk.partial + int64_t(team) * pk.partial_per_team;
    const int num_items = VOXEL ? va.num_items : pa.num_items;
    const int mm = pk.mm;
    if constexpr (VOXEL) {
        team_query_table(QT, va, MC, tid, PNT);
    }
    volatile int* slot = pk.slots + team;
    bool first = true;
    for (;;) {
        if (crank == 0 && tid == 0) {
            *slot = first ? team : nteams + atomicAdd(pk.queue, 1);
            __threadfence();
        }
        first = false;
        team_sync(C);
        const int it = *slot;
        if (it >= num_items) break;

        // ---- stage the training set (every CTA of the team)
        int n, m, s, vid = 0;
        int64_t qo = 0;
        double lam, jitter, mean_f = 0.0;
        int kind;
        VoxelCtx vc{};
        if constexpr (VOXEL) {
            vc = team_stage_voxel(va, it, X, F, NZ, NP, tid, PNT);
            s = vc.s;
            vid = vc.vid;
            n = vc.n;
            mean_f = vc.mean_f;
            m = va.M;
            lam = va.lam;
            jitter = va.jitter;
            kind = va.kernel;
            team_grid_coords(GC, vc, mm, tid);
        } else {
            s = pa.items[it];
            const int64_t xo = pa.x_off[s];
            qo = pa.q_off[s];
            n = int(pa.x_off[s + 1] - xo);
            m = int(pa.q_off[s + 1] - qo);
            lam = pa.lam[s];
            jitter = pa.jitter;
            kind = pa.kernel;
            for (int r = tid; r < NP; r += PNT) {
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
        __syncthreads();
        const int n32 = round_up(n, PNB);
        const int A32 = round_up(m + 1, PNB);
        const int R = n32 + A32;
        const int np = n32 / PNB;

        // M(r, c), c < n32 (only r >= c is used for r < n32)
        auto mval = [&](int r, int c, double jit) -> double {
            if (r < n32) {
                if (r == c) {
                    if (r >= n) return 1.0;
                    double dg = xadd(1.0, NZ[r]);
                    return jit != 0.0 ? xadd(dg, jit) : dg;
                }
                if (r >= n || c >= n) return 0.0;
                return kernel_value(kind, lam, dist2_exact(X[2 * r], X[2 * r + 1], X[2 * c], X[2 * c + 1]));
            }
            const int q = r - n32;
            if (c >= n || q > m) return 0.0;
            if (q == 0) return F[c];
            double g0, g1;
            if constexpr (VOXEL) {
                const int qt = QT[q];
                g0 = GC[qt & 0xffff];
                g1 = GC[mm + (qt >> 16)];
            } else {
                g0 = pa.xs[(qo + q - 1) * 2];
                g1 = pa.xs[(qo + q - 1) * 2 + 1];
            }
            return kernel_value(kind, lam, dist2_exact(X[2 * c], X[2 * c + 1], g0, g1));
        };

        bool ok = false;
        // ---- GEMM waves: P_pt (+)= M / - sum_{q in [q0, q1)} L[jt:, q-block] L[jt:jt+32, q-block]^T
        // over 16x32 row tiles (two 8-row x four 8-column DMMA tiles per warp), in
        // waves of one tile per participating warp of the team (warps w0..PW-1 of
        // every CTA).  The B operand block L[jt:jt+32, 32q:32q+32] is staged once
        // per CTA in shared memory by cp.async (double-buffered one block ahead);
        // each warp's A fragments of block q+1 load into registers while block q's
        // 64 DMMAs issue.  init: 0 -> M (generated), 1 -> P_pt from the workspace.
        auto gemm_waves = [&](int pt, int q0, int q1, int init, int w0, double jit) {
            const int jt = pt * PNB;
            double* Pt = Lw + panel_base(R, pt);
            const int ldt = R - jt;
            const int T = (R - jt) / PRT;
            const int wpc = PW - w0;                    // participating warps per CTA
            const int nw = C * wpc;
            const int gw = (crank * wpc + (warp - w0) + pt) % nw;
            const int waves = (T + nw - 1) / nw;
            const int nthr = wpc * 32, ltid = tid - w0 * 32;
            auto bar = [&]() {
                if (w0 == 0) __syncthreads();
                else asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
            };
            for (int w = 0; w < waves; ++w) {
                const int t = w * nw + gw;
                const bool act = t < T;
                const int r0 = jt + (act ? t : 0) * PRT;
                double acc[2][4][2];
                double* dst = Pt + (r0 - jt) + g;
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            double v = 0.0;
                            if (act)
                                v = init ? __ldcg(dst + int64_t(8 * b + 2 * tig + e) * ldt + 8 * a)
                                         : mval(r0 + 8 * a + g, jt + 8 * b + 2 * tig + e, jit);
                            acc[a][b][e] = -v;        // accumulate -P: the fragments stay un-negated

                        }
                if (q1 > q0) {
                    auto stage_b = [&](int q) {
                        const int ldq = R - q * PNB;
                        const double* src = Lw + panel_base(R, q) + (jt - q * PNB);
                        double* bdst = BS + (q & 1) * (PNB * PLD);
                        for (int e = ltid; e < PNB * 8; e += nthr) {
                            const int k = e >> 3, r = (e & 7) * 4;
                            cp_async16(bdst + k * PLD + r, src + int64_t(k) * ldq + r);
                            cp_async16(bdst + k * PLD + r + 2, src + int64_t(k) * ldq + r + 2);
                        }
                        cp_async_commit();
                    };
                    auto load_a = [&](int q, double (&f)[2][8]) {
                        const int ldq = R - q * PNB;
                        const double* src = Lw + panel_base(R, q) + int64_t(tig) * ldq +
                                            (r0 - q * PNB) + g;
#pragma unroll
                        for (int st = 0; st < 8; ++st)
#pragma unroll
                            for (int a = 0; a < 2; ++a)
                                f[a][st] = act ? __ldcg(src + int64_t(4 * st) * ldq + 8 * a) : 0.0;
                    };
                    double fa[2][8], na[2][8];
                    stage_b(q0);
                    load_a(q0, fa);
                    for (int q = q0; q < q1; ++q) {
                        cp_async_wait_all();
                        bar();                        // BS[q & 1] complete; BS[(q+1) & 1] free
                        if (q + 1 < q1) {
                            stage_b(q + 1);
                            load_a(q + 1, na);
                        }
                        const double* bs = BS + (q & 1) * (PNB * PLD) + tig * PLD + g;
                        if (act)
#pragma unroll
                        for (int st = 0; st < 8; ++st) {
                            double fb[4];
#pragma unroll
                            for (int b = 0; b < 4; ++b) fb[b] = bs[4 * st * PLD + 8 * b];
#pragma unroll
                            for (int a = 0; a < 2; ++a)
#pragma unroll
                                for (int b = 0; b < 4; ++b)
                                    dmma_acc(acc[a][b][0], acc[a][b][1], fa[a][st], fb[b]);
                        }
                        if (q + 1 < q1) {
#pragma unroll
                            for (int st = 0; st < 8; ++st) {
                                fa[0][st] = na[0][st];
                                fa[1][st] = na[1][st];
                            }
                        }
                    }
                    bar();                            // BS reads done before the next wave
                }
                if (act) {
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
#pragma unroll
                            for (int e = 0; e < 2; ++e)
                                __stcg(dst + int64_t(8 * b + 2 * tig + e) * ldt + 8 * a, -acc[a][b][e]);
                }
            }
        };

        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            const double jit = attempt ? jitter : 0.0;
            ok = true;
#ifdef VX_PHASE_TIMING
            long long tph = clock64();
#endif
            // Look-ahead (teams of several CTAs, the latency regime): the bulk of
            // panel p+1's update (A1, blocks < p) runs during panel p's diagonal
            // chain and only the last block (A2) stays on the critical path.  One-CTA
            // teams (the throughput regime, two CTAs per SM) update each panel in
            // one pass with all warps: the other CTA of the SM covers the chain, and
            // the look-ahead's extra pass over P and its 7-warp waves cost more.
            const bool ahead = C > 1;
            if (ahead) {                              // P_0 = M[:, 0:32]
                gemm_waves(0, 0, 0, 0, 0, jit);
                team_sync(C);
            }
            for (int p = 0; p < np; ++p) {
                const int j = p * PNB;
                double* Pp = Lw + panel_base(R, p);
                const int ldp = R - j;
                // ---- (A) P_p = M - L[j:, :j] L[j:j+32, :j]^T; with look-ahead only the
                // last finished panel p-1 remains (A2), the earlier blocks were applied
                // by (A1) during panel p-1's diagonal chain
                if (!ahead || p > 0) {
                    if (ahead) gemm_waves(p, p - 1, p, 1, 0, jit);
                    else gemm_waves(p, 0, p, 0, 0, jit);
                    VX_PHASE(12, tph);                // phase A / A2
                    team_sync(C);
                    VX_PHASE(13, tph);                // team barrier after A
                }
                // ---- (D) warp 0 of every CTA factors the diagonal block (redundantly:
                // every CTA takes the same pivot decision) while warps 1..7 run (A1),
                // the look-ahead: P_{p+1} = M - (blocks 0 .. p-1), which do not depend
                // on panel p
                if (warp == 0) {
                    const bool good = diag_block_factor(Pp, ldp, LD, LI, smem + lay.DINV, lane);
                    if (lane == 0) smem[lay.FLAG] = good ? 1.0 : 0.0;
                } else if (ahead && p + 1 < np) {
                    gemm_waves(p + 1, 0, p, 0, 1, jit);
                }
                __syncthreads();
                VX_PHASE(14, tph);                    // diagonal || look-ahead
                if (smem[lay.FLAG] == 0.0) {          // the same decision in every CTA
                    ok = false;
                    team_sync(C);
                    break;
                }
                // ---- (B) L[j+32:, j:j+32] = P[32:] L_dd^-T, blockwise by 8 columns with
                // DMMA: X_kb = (P_kb - sum_{i<kb} X_i L_{kb,i}^T) D_kb^-T, D_kb^-1 the
                // 8x8 diagonal-block inverses (no off-diagonal inverse on the chain).
                // Accumulators (C layout) become A operands by two shuffles per value.
                const int T2 = (R - j) / PRT - PNB / PRT;
                const int nw = C * PW;
                const int gw = (crank * PW + warp + p) % nw;
                // A fragment (k-chunk sl) of an 8x8 C-layout block held as (c0, c1)
                auto c_to_a = [&](double c0, double c1, int sl) {
                    const int srcl = g * 4 + 2 * sl + (tig >> 1);
                    const double v0 = __shfl_sync(FULL, c0, srcl);
                    const double v1 = __shfl_sync(FULL, c1, srcl);
                    return (tig & 1) ? v1 : v0;
                };
                for (int t = gw; t < T2; t += nw) {
                    double* src = Pp + PNB + t * PRT + g;
                    double pc[2][4][2];
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
#pragma unroll
                            for (int e = 0; e < 2; ++e)
                                pc[a][b][e] = __ldcg(src + int64_t(8 * b + 2 * tig + e) * ldp + 8 * a);
                    double xa[2][4][2];       // X_i as A fragments (k-chunks 0, 1)
#pragma unroll
                    for (int kb = 0; kb < 4; ++kb) {
#pragma unroll
                        for (int a = 0; a < 2; ++a) {
                            double c0 = pc[a][kb][0], c1 = pc[a][kb][1];
#pragma unroll
                            for (int i = 0; i < kb; ++i)
#pragma unroll
                                for (int sl = 0; sl < 2; ++sl)
                                    dmma_acc(c0, c1, -xa[a][i][sl],
                                             LD[(8 * kb + g) * PLDL + 8 * i + 4 * sl + tig]);
                            // X = C D^-T: B[q][c] = D^-1[c][q]
                            double d0 = 0.0, d1 = 0.0;
#pragma unroll
                            for (int sl = 0; sl < 2; ++sl)
                                dmma_acc(d0, d1, c_to_a(c0, c1, sl),
                                         LI[(8 * kb + g) * PLD + 8 * kb + 4 * sl + tig]);
                            pc[a][kb][0] = d0;
                            pc[a][kb][1] = d1;
                            if (kb < 3) {
#pragma unroll
                                for (int sl = 0; sl < 2; ++sl) xa[a][kb][sl] = c_to_a(d0, d1, sl);
                            }
                        }
                    }
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
#pragma unroll
                            for (int e = 0; e < 2; ++e)
                                __stcg(src + int64_t(8 * b + 2 * tig + e) * ldp + 8 * a, pc[a][b][e]);
                }
                VX_PHASE(15, tph);                    // phase B triangular update
                team_sync(C);
                VX_PHASE(16, tph);                    // team barrier after B
            }
        }
        if (!ok) {
            if (crank == 0 && tid == 0) {
                if constexpr (VOXEL) {
                    va.cand_status[s] = VX_ST_CHOL_FAIL;
                    const uint8_t st = va.state[vid];
                    va.cand_before[s] = st;
                    va.cand_after[s] = st;
                } else {
                    pa.status[s] = VX_ST_CHOL_FAIL;
                }
            }
            continue;       // the next item's slot write follows a team barrier
        }
        // ---- epilogue (1): per-warp partial sums over the team's panels
        //   ss_q = sum_k W(q, k)^2, dz_q = sum_k W(q, k) W(0, k), aug row q = n32 + q
        {
            const int nw = C * PW;
            const int gw = crank * PW + warp;
            double* mine = part + int64_t(gw) * 2 * A32;
            for (int q0 = 0; q0 < A32; q0 += 32) {
                const int q = q0 + lane;
                double ss0 = 0.0, ss1 = 0.0, dz0 = 0.0, dz1 = 0.0;
                for (int p = gw; p < np; p += nw) {
                    const int ldp = R - p * PNB;
                    const double* col = Lw + panel_base(R, p) + (n32 - p * PNB);
#pragma unroll 4
                    for (int c = 0; c < PNB; c += 2) {
                        const double w0 = __ldcg(col + int64_t(c) * ldp + q);
                        const double w1 = __ldcg(col + int64_t(c + 1) * ldp + q);
                        const double z0 = __ldcg(col + int64_t(c) * ldp);
                        const double z1 = __ldcg(col + int64_t(c + 1) * ldp);
                        ss0 = fma(w0, w0, ss0);
                        ss1 = fma(w1, w1, ss1);
                        dz0 = fma(w0, z0, dz0);
                        dz1 = fma(w1, z1, dz1);
                    }
                }
                mine[q] = ss0 + ss1;
                mine[A32 + q] = dz0 + dz1;
            }
        }
        team_sync(C);
        // ---- epilogue (2): team rank 0 reduces in a fixed order and finishes the voxel
        if (crank == 0) {
            const int nw = C * PW;
            double* MU = smem + lay.MU;
            double* VAR = smem + lay.VAR;
            for (int c = tid + 1; c <= m; c += PNT) {
                double ss = 0.0, mu = 0.0;
                for (int w = 0; w < nw; ++w) {
                    ss += __ldcg(part + int64_t(w) * 2 * A32 + c);
                    mu += __ldcg(part + int64_t(w) * 2 * A32 + A32 + c);
                }
                const double var = 1.0 - ss;
                if constexpr (VOXEL) {
                    MU[c] = xadd(mu, mean_f);
                    VAR[c] = var < 0.0 ? 0.0 : var;
                } else {
                    pa.mu[qo + c - 1] = mu;
                    pa.var[qo + c - 1] = var;
                }
            }
            __syncthreads();
            if constexpr (VOXEL) {
                team_voxel_epilogue(va, vc, X, GC, QT, mm, MU, VAR, smem + lay.COL, tid, PNT);
            } else {
                if (tid == 0) pa.status[s] = VX_ST_OK;
            }
        }
        // the partial sums are rewritten by the next item only after its
        // staging barrier (team_sync at the top of the loop)
    }
}
