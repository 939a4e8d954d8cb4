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
    int X, F, NZ, GC, QT, LD, LI, MU, VAR, COL, FLAG, total;
    __host__ __device__ PanelLayout(int np32, int mcols, int mmax) {
        int o = 0;
        X = o; o += 2 * np32;
        F = o; o += np32;
        NZ = o; o += np32;
        GC = o; o += 2 * MAX_MM;
        QT = o; o += mcols / 2 + 1;       // int32 (ri | si << 16) per column
        LD = o; o += PNB * PLD;           // factored diagonal block (row-major)
        LI = o; o += PNB * PLD;           // its inverse (row-major)
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

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
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
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
            const double jit = attempt ? jitter : 0.0;
            ok = true;
            for (int p = 0; p < np; ++p) {
                const int j = p * PNB;
                double* Pp = Lw + panel_base(R, p);
                const int ldp = R - j;
                // ---- phase A: P = M[j:, j:j+32] - L[j:, :j] L[j:j+32, :j]^T in 16x32
                // row tiles (two 8-row DMMA tiles x four 8-column tiles per warp)
                const int T = (R - j) / PRT;
                const int nw = C * PW;
                const int gw = (crank * PW + warp + p) % nw;
                for (int t = gw; t < T; t += nw) {
                    const int r0 = j + t * PRT;
                    double acc[2][4][2];
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
#pragma unroll
                            for (int e = 0; e < 2; ++e)
                                acc[a][b][e] = mval(r0 + 8 * a + g, j + 8 * b + 2 * tig + e, jit);
                    // k runs over the finished panels q < p (columns 32q .. 32q+31);
                    // software-pipelined: the fragments of step s+1 load while the
                    // DMMAs of step s issue
                    const int steps = p * (PNB / 4);
                    auto frag_ptr = [&](int st, int row0) {
                        const int q = st >> 3, kk = (st & 7) * 4;
                        const int ldq = R - q * PNB;
                        return Lw + panel_base(R, q) + int64_t(kk + tig) * ldq + (row0 - q * PNB) + g;
                    };
                    double fa[2], fb[4];
                    if (steps > 0) {
                        const double* pa_ = frag_ptr(0, r0);
                        const double* pb_ = frag_ptr(0, j);
                        fa[0] = __ldcg(pa_);
                        fa[1] = __ldcg(pa_ + 8);
#pragma unroll
                        for (int b = 0; b < 4; ++b) fb[b] = __ldcg(pb_ + 8 * b);
                    }
                    for (int st = 0; st < steps; ++st) {
                        double na[2] = {0.0, 0.0}, nb[4] = {0.0, 0.0, 0.0, 0.0};
                        if (st + 1 < steps) {
                            const double* pa_ = frag_ptr(st + 1, r0);
                            const double* pb_ = frag_ptr(st + 1, j);
                            na[0] = __ldcg(pa_);
                            na[1] = __ldcg(pa_ + 8);
#pragma unroll
                            for (int b = 0; b < 4; ++b) nb[b] = __ldcg(pb_ + 8 * b);
                        }
#pragma unroll
                        for (int a = 0; a < 2; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b) dmma_acc(acc[a][b][0], acc[a][b][1], -fa[a], fb[b]);
                        fa[0] = na[0];
                        fa[1] = na[1];
#pragma unroll
                        for (int b = 0; b < 4; ++b) fb[b] = nb[b];
                    }
                    double* dst = Pp + (r0 - j) + g;
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
#pragma unroll
                            for (int e = 0; e < 2; ++e)
                                __stcg(dst + int64_t(8 * b + 2 * tig + e) * ldp + 8 * a, acc[a][b][e]);
                }
                team_sync(C);
                // ---- phase B (1): every CTA factors the diagonal block (warp 0).
                // Left-looking, row r by lane r, rows in shared memory (LD, stride
                // PLDL: conflict-free row reads); then column c of L_dd^-1 by lane c
                // into LI (row-major).  A pivot that is not > 0 fails (dpotrf).
                if (warp == 0) {
                    double* myrow = LD + lane * PLDL;
#pragma unroll 4
                    for (int c = 0; c < PNB; ++c) myrow[c] = __ldcg(Pp + int64_t(c) * ldp + lane);
                    __syncwarp();
                    bool good = true;
                    for (int c = 0; c < PNB; ++c) {
                        const double* rowc = LD + c * PLDL;
                        double s0 = myrow[c], s1 = 0.0;
                        int k = 0;
                        for (; k + 1 < c; k += 2) {
                            s0 = fma(-myrow[k], rowc[k], s0);
                            s1 = fma(-myrow[k + 1], rowc[k + 1], s1);
                        }
                        if (k < c) s0 = fma(-myrow[k], rowc[k], s0);
                        const double sc = s0 + s1;
                        const double piv = __shfl_sync(FULL, sc, c);
                        if (!(piv > 0.0)) good = false;
                        const double d = sqrt(piv);
                        __syncwarp();
                        myrow[c] = lane == c ? d : (lane > c ? sc / d : 0.0);
                        __syncwarp();
                    }
                    // x = column `lane` of L_dd^-1: x_r = (e_r - sum_{k<r} L(r,k) x_k) / L(r,r)
                    for (int r = 0; r < PNB; ++r) {
                        const double* rowr = LD + r * PLDL;
                        double s0 = (r == lane) ? 1.0 : 0.0, s1 = 0.0;
                        int k = lane;                      // x_k = 0 for k < lane
                        for (; k + 1 < r; k += 2) {
                            s0 = fma(-rowr[k], LI[k * PLD + lane], s0);
                            s1 = fma(-rowr[k + 1], LI[(k + 1) * PLD + lane], s1);
                        }
                        if (k < r) s0 = fma(-rowr[k], LI[k * PLD + lane], s0);
                        LI[r * PLD + lane] = r < lane ? 0.0 : (s0 + s1) / rowr[r];
                    }
                    if (lane == 0) smem[lay.FLAG] = good ? 1.0 : 0.0;
                }
                __syncthreads();
                if (smem[lay.FLAG] == 0.0) {      // the same decision in every CTA
                    ok = false;
                    team_sync(C);
                    break;
                }
                // ---- phase B (2): L[j+32:, j:j+32] = P[32:] L_dd^-T (DMMA with L_dd^-1)
                const int T2 = T - PNB / PRT;
                for (int t = gw; t < T2; t += nw) {
                    double* src = Pp + PNB + t * PRT + g;
                    double fa2[2][8];
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int kc = 0; kc < 8; ++kc)
                            fa2[a][kc] = __ldcg(src + int64_t(4 * kc + tig) * ldp + 8 * a);
                    double acc[2][4][2];
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
                    for (int kc = 0; kc < 8; ++kc) {
                        double fb[4];
#pragma unroll
                        for (int b = 0; b < 4; ++b) fb[b] = LI[(8 * b + g) * PLD + 4 * kc + tig];
#pragma unroll
                        for (int a = 0; a < 2; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b) dmma_acc(acc[a][b][0], acc[a][b][1], fa2[a][kc], fb[b]);
                    }
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b)
#pragma unroll
                            for (int e = 0; e < 2; ++e)
                                __stcg(src + int64_t(8 * b + 2 * tig + e) * ldp + 8 * a, acc[a][b][e]);
                }
                team_sync(C);
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
