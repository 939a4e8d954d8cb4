// Device-resident voxel map: hashing, per-voxel point arena, lifecycle, and
// the densify / Gaussian-init orchestration (voxel_map.py:268-355,
// gpr.py:269-311, pipeline.py:139-171).
//
// HBM layout (all SoA, grown by doubling on demand):
//   hash table     tcap slots: packed key (u64), voxel id (i32), first-touch
//                  stamp (u64), frame rank (i32); open addressing, linear probe
//   voxel records  V: key (3 x i64), state (u8), value axis (i8), raw count
//                  (i32), raw offset (i64), raw capacity (i32), prediction
//                  slot (i32), has-prediction (u8)
//   point arena    rows of xyz (3 x f64) and rgb (3 x f64); each voxel owns a
//                  contiguous run that doubles (relocating) when full, so a
//                  solve reads its raw points with unit stride; raw noise is
//                  sensor_var for every raw point and is not stored
//   predictions    slots x M (M = (n_s n_r)^2): xyz, rgb, clipped variance —
//                  the last prediction of a voxel and the pseudo-observations
//                  of its next solve (voxel_map.py:257-259)
//
// store_frame reproduces the reference's observable order exactly:
//   first-touch order of the touched keys = order of each key's smallest point
//   index (np.unique return_index + stable argsort, voxel_map.py:324-326),
//   computed as an atomicMin of (frame stamp, index) per slot and a scan of
//   "is first point" flags; points of a voxel keep frame order (the boolean
//   mask at line 330) by a stable radix sort of (rank, index) pairs.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>

#include "vx_common.cuh"
#include "vx_internal.h"

struct VxMap {
    VxMapConfig cfg;
    int M = 0;
    int64_t frame_index = -1;
    uint32_t epoch = 0;
    // hash table
    int64_t tcap = 0;
    vx::DevBuf tkeys, tvals, tfirst, trank;
    // voxels
    int64_t num_voxels = 0, vcap = 0;
    vx::DevBuf keys3, pkey, state, axis, raw_count, raw_off, raw_cap, pred_slot, has_pred, last_first;
    // arena
    int64_t arena_top = 0, arena_cap = 0;
    vx::DevBuf axyz, argb;
    // predictions
    int64_t num_slots = 0, slot_cap = 0;
    vx::DevBuf pxyz, prgb, pvar;
    // frame scratch (per point)
    vx::DevBuf pslot, flags, fscan, prank, pidx, prank2, pidx2;
    // frame scratch (per touched voxel)
    vx::DevBuf tslot, tcnt, tseg, tnew, tnewscan, tneed, tneedscan, tbase, treloc, frame_vids, fb, fa;
    int64_t frame_touched = 0;
    // densify
    vx::DevBuf cflag, cscan, cand_voxel, cand_n, cand_status, cand_before, cand_after, items,
        okflag, okscan, solved_vids, cand_axis, cand_meanf;
    int64_t solve_candidates = 0, solved = 0;
    int64_t first_count = 0;   // first solves of the last ingest, listed in `items`
    // counters (device) + pinned mirror
    vx::DevBuf counters;
    int64_t* host_counters = nullptr;      // mapped pinned memory (see read_counters)
    int64_t* host_counters_dev = nullptr;  // its device alias
    // temporaries
    vx::DevBuf scan_tmp, sort_tmp, gpr_work, gpr_work2, stage;
    // small frames: the size buckets run concurrently on their own streams
    cudaStream_t bstream[8] = {};
    cudaEvent_t bfork = nullptr, bdone[8] = {};
};

namespace vx {

// counters layout (int64)
enum {
    C_ERR = 0,        // bit 1: non-finite, bit 2: out of lattice range, bit 4: table full
    C_INSERTED,       // new table entries this frame
    C_U,              // touched voxels
    C_NEW,            // new voxels
    C_NEED,           // arena rows to allocate
    C_KEPT,           // points kept by this shard
    C_READY,          // UNREADY->READY transitions
    C_S,              // densify candidates
    C_MAXN,
    C_NEWSLOTS,
    C_B0, C_B1, C_B2, C_B3, C_B4, C_B5, C_B6, C_B7,   // bucket counts
    C_F0, C_F1, C_F2, C_F3, C_F4, C_F5, C_F6, C_F7,   // bucket fill cursors
    C_O0, C_O1, C_O2, C_O3, C_O4, C_O5, C_O6, C_O7,   // bucket bases
    C_OK, C_DEGEN, C_CHOL, C_FIRST, C_CONV,
    C_MAXSEG,         // longest per-voxel run of this frame's points
    C_BIG,            // runs longer than SEG_WARP_MAX (segment-append big list)
    C_COUNT
};

// ------------------------------------------------------------------ kernels
__global__ void k_fill_u64(uint64_t* p, int64_t n, uint64_t v) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__device__ __forceinline__ uint32_t shard_of(uint64_t pk, int world) {
    return uint32_t(mix64(pk ^ 0x9e3779b97f4a7c15ull) % uint64_t(world));
}

// H1 + table insert: key = floor(p / voxel_size) (voxel_map.py:143)
__global__ void k_hash_points(const double* __restrict__ xyz, int64_t n, double vs,
                              uint64_t* tkeys, uint64_t* tfirst, int64_t tmask, uint32_t epoch,
                              int rank, int world, int32_t* pslot, long long* ctr) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = xyz[i * 3], y = xyz[i * 3 + 1], z = xyz[i * 3 + 2];
    pslot[i] = -1;
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) {
        atomicOr(reinterpret_cast<unsigned long long*>(ctr + C_ERR), 1ull);
        return;
    }
    const double fx = floor(xdiv(x, vs)), fy = floor(xdiv(y, vs)), fz = floor(xdiv(z, vs));
    const double lim = double(KEY_LIM);   // representable keys: [-2^20, 2^20)
    if (!(fx >= -lim && fx < lim && fy >= -lim && fy < lim && fz >= -lim && fz < lim)) {
        atomicOr(reinterpret_cast<unsigned long long*>(ctr + C_ERR), 2ull);
        return;
    }
    const uint64_t pk = pack_key(int64_t(fx), int64_t(fy), int64_t(fz));
    if (world > 1 && shard_of(pk, world) != uint32_t(rank)) return;
    uint64_t h = mix64(pk) & uint64_t(tmask);
    for (int64_t probe = 0;; ++probe) {
        if (probe > 256 || probe > tmask) {      // table too full: host grows + retries
            atomicOr(reinterpret_cast<unsigned long long*>(ctr + C_ERR), 4ull);
            return;
        }
        uint64_t cur = tkeys[h];
        if (cur == pk) break;
        if (cur == EMPTY_KEY) {
            uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(tkeys + h),
                                      (unsigned long long)EMPTY_KEY, (unsigned long long)pk);
            if (prev == EMPTY_KEY) break;
            if (prev == pk) break;
        }
        h = (h + 1) & uint64_t(tmask);
    }
    pslot[i] = int32_t(h);
    const uint64_t stamp = (uint64_t(0xffffffffu - epoch) << 32) | uint64_t(uint32_t(i));
    atomicMin(reinterpret_cast<unsigned long long*>(tfirst + h), (unsigned long long)stamp);
}

__global__ void k_first_flags(const int32_t* pslot, const uint64_t* tfirst, int64_t n,
                              int32_t* flags) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t s = pslot[i];
    flags[i] = (s >= 0 && uint32_t(tfirst[s]) == uint32_t(i)) ? 1 : 0;
}

__global__ void k_rank_slots(const int32_t* pslot, const int32_t* flags, const int32_t* fscan,
                             int64_t n, int32_t* trank, int32_t* tslot, int32_t* tcnt) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n || !flags[i]) return;
    const int32_t r = fscan[i];
    tslot[r] = pslot[i];
    trank[pslot[i]] = r;
    tcnt[r] = 0;
}

// rank of each point's voxel in first-touch order (U: not kept) and an
// ordinal among the frame's points of that voxel (atomic, arbitrary order:
// the segment-append kernels restore index order)
__global__ void k_point_rank(const int32_t* pslot, const int32_t* trank, int64_t n, uint32_t U,
                             uint32_t* prank, uint32_t* pord, int32_t* tcnt) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t s = pslot[i];
    uint32_t r = U, o = 0;
    if (s >= 0) {
        r = uint32_t(trank[s]);
        o = uint32_t(atomicAdd(tcnt + r, 1));
    }
    prank[i] = r;
    if (pord) pord[i] = o;
}

// counting placement: point i goes to slot tseg[r] + ordinal of its voxel run
__global__ void k_place(const uint32_t* prank, const uint32_t* pord, int64_t n, uint32_t U,
                        const int32_t* tseg, uint32_t* sidx) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = prank[i];
    if (r < U) sidx[int64_t(tseg[r]) + pord[i]] = uint32_t(i);
}

// Segment append (replaces the stable radix sort of (rank, index) pairs and
// the per-point append): each voxel run of sidx holds its frame indices in
// arbitrary order; sorting the run restores frame order (voxel_map.py:331-336
// appends points in frame order), then the run's rows are gathered from the
// frame and written contiguously to the voxel's arena run.
constexpr int SEG_WARP_MAX = 512;     // runs a warp sorts in its shared-memory slice
constexpr int SEG_BIG_MAX = 8192;     // runs a CTA sorts (longer: radix-sort fallback)

__device__ __forceinline__ void seg_copy_rows(const double* __restrict__ xyz,
                                              const double* __restrict__ rgb, int64_t i,
                                              int64_t dst, double* axyz, double* argb) {
    const double x0 = xyz[i * 3], x1 = xyz[i * 3 + 1], x2 = xyz[i * 3 + 2];
    const double c0 = rgb[i * 3], c1 = rgb[i * 3 + 1], c2 = rgb[i * 3 + 2];
    axyz[dst * 3] = x0;
    axyz[dst * 3 + 1] = x1;
    axyz[dst * 3 + 2] = x2;
    argb[dst * 3] = c0;
    argb[dst * 3 + 1] = c1;
    argb[dst * 3 + 2] = c2;
}

// bitonic sort of P (power of two) keys in shared memory by `nt` threads
__device__ __forceinline__ void bitonic_smem(uint32_t* a, int P, int t, int nt, bool warp) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int q = t; q < P / 2; q += nt) {
                const int i = 2 * j * (q / j) + (q % j), l = i + j;
                const uint32_t x = a[i], y = a[l];
                const bool asc = (i & k) == 0;
                if ((x > y) == asc) {
                    a[i] = y;
                    a[l] = x;
                }
            }
            if (warp) __syncwarp(); else __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(256) k_seg_append_warp(
        const uint32_t* sidx, const int32_t* tseg, const int32_t* tcnt, int64_t U,
        const int32_t* tbase, const int32_t* frame_vids, const int64_t* raw_off,
        const double* __restrict__ xyz, const double* __restrict__ rgb, double* axyz,
        double* argb, int32_t* big, long long* ctr) {
    __shared__ uint32_t sm[8][SEG_WARP_MAX];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* a = sm[w];
    const int64_t nw = int64_t(gridDim.x) * 8;
    for (int64_t r = int64_t(blockIdx.x) * 8 + w; r < U; r += nw) {
        const int L = tcnt[r];
        if (L <= 0) continue;
        const int64_t s0 = tseg[r];
        const int64_t dst = raw_off[frame_vids[r]] + tbase[r];
        if (L <= 32) {
            uint32_t v = lane < L ? sidx[s0 + lane] : 0xffffffffu;
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1) {
                    const uint32_t o = __shfl_xor_sync(FULL, v, j);
                    const bool up = (lane & k) == 0, low = (lane & j) == 0;
                    v = (low == up) ? (v < o ? v : o) : (v > o ? v : o);
                }
            }
            if (lane < L) seg_copy_rows(xyz, rgb, v, dst + lane, axyz, argb);
        } else if (L <= SEG_WARP_MAX) {
            int P = 64;
            while (P < L) P <<= 1;
            for (int q = lane; q < P; q += 32) a[q] = q < L ? sidx[s0 + q] : 0xffffffffu;
            __syncwarp();
            bitonic_smem(a, P, lane, 32, true);
            for (int q = lane; q < L; q += 32) seg_copy_rows(xyz, rgb, a[q], dst + q, axyz, argb);
            __syncwarp();
        } else if (lane == 0) {
            big[atomicAdd(reinterpret_cast<unsigned long long*>(ctr + C_BIG), 1ull)] = int32_t(r);
        }
    }
}

__global__ void __launch_bounds__(1024) k_seg_append_big(
        const uint32_t* sidx, const int32_t* tseg, const int32_t* tcnt, const int32_t* tbase,
        const int32_t* frame_vids, const int64_t* raw_off, const double* __restrict__ xyz,
        const double* __restrict__ rgb, double* axyz, double* argb, const int32_t* big,
        const long long* ctr) {
    __shared__ uint32_t a[SEG_BIG_MAX];
    const long long nbig = ctr[C_BIG];
    for (long long b = blockIdx.x; b < nbig; b += gridDim.x) {
        const int r = big[b];
        const int L = tcnt[r];
        const int64_t s0 = tseg[r];
        const int64_t dst = raw_off[frame_vids[r]] + tbase[r];
        int P = 1024;
        while (P < L) P <<= 1;
        for (int q = threadIdx.x; q < P; q += blockDim.x) a[q] = q < L ? sidx[s0 + q] : 0xffffffffu;
        __syncthreads();
        bitonic_smem(a, P, threadIdx.x, blockDim.x, false);
        for (int q = threadIdx.x; q < L; q += blockDim.x) seg_copy_rows(xyz, rgb, a[q], dst + q, axyz, argb);
        __syncthreads();
    }
}

__device__ __forceinline__ int32_t grow_cap(int64_t need) {
    int64_t c = 16;
    while (c < need) c *= 2;
    return int32_t(c);
}

__global__ void k_touched_prep(const int32_t* tslot, const int32_t* tcnt, int64_t U,
                               const int32_t* tvals, const int32_t* raw_count, const int32_t* raw_cap,
                               int32_t* tnew, int64_t* tneed, long long* maxseg) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= U) return;
    const int32_t vid = tvals[tslot[r]];
    const bool isnew = vid < 0;
    tnew[r] = isnew ? 1 : 0;
    const int64_t cnt0 = isnew ? 0 : raw_count[vid];
    const int64_t cap0 = isnew ? 0 : raw_cap[vid];
    const int64_t want = cnt0 + tcnt[r];
    tneed[r] = want > cap0 ? int64_t(grow_cap(want)) : 0;
    if (tcnt[r] > SEG_WARP_MAX) atomicMax(reinterpret_cast<unsigned long long*>(maxseg), (unsigned long long)tcnt[r]);
}

struct CommitArgs {
    const int32_t* tslot;
    const int32_t* tnewscan;
    const int32_t* tnew;
    const int64_t* tneed;
    const int64_t* tneedscan;
    int64_t U;
    int64_t num_voxels;
    int64_t arena_top;
    const uint64_t* tkeys;
    int32_t* tvals;
    int64_t* keys3;
    uint64_t* pkey;
    uint8_t* state;
    int8_t* axis;
    int32_t* raw_count;
    int64_t* raw_off;
    int32_t* raw_cap;
    int32_t* pred_slot;
    uint8_t* has_pred;
    int32_t* frame_vids;
    int32_t* last_first;
    const uint64_t* tfirst;
    uint8_t* fb;
    int32_t* tbase;
    int64_t* treloc;
};

__global__ void k_touched_commit(CommitArgs a) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= a.U) return;
    const int32_t slot = a.tslot[r];
    int32_t vid;
    if (a.tnew[r]) {
        vid = int32_t(a.num_voxels + a.tnewscan[r]);
        a.tvals[slot] = vid;
        const uint64_t pk = a.tkeys[slot];
        int64_t k0, k1, k2;
        unpack_key(pk, &k0, &k1, &k2);
        a.keys3[int64_t(vid) * 3] = k0;
        a.keys3[int64_t(vid) * 3 + 1] = k1;
        a.keys3[int64_t(vid) * 3 + 2] = k2;
        a.pkey[vid] = pk;
        a.state[vid] = VX_UNREADY;
        a.axis[vid] = -1;
        a.raw_count[vid] = 0;
        a.raw_off[vid] = 0;
        a.raw_cap[vid] = 0;
        a.pred_slot[vid] = -1;
        a.has_pred[vid] = 0;
    } else {
        vid = a.tvals[slot];
    }
    a.frame_vids[r] = vid;
    a.last_first[vid] = int32_t(uint32_t(a.tfirst[slot]));   // first point of this frame
    a.fb[r] = a.state[vid];
    a.tbase[r] = a.raw_count[vid];
    a.treloc[r] = -1;
    if (a.tneed[r] > 0) {
        if (a.raw_count[vid] > 0) a.treloc[r] = a.raw_off[vid];
        a.raw_off[vid] = a.arena_top + a.tneedscan[r];
        a.raw_cap[vid] = int32_t(a.tneed[r]);
    }
}

// move a relocated voxel's existing points to its new run (warp per voxel)
__global__ void k_relocate(const int64_t* treloc, const int32_t* frame_vids, const int32_t* tbase,
                           int64_t U, const int64_t* raw_off, double* axyz, double* argb) {
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= U) return;
    const int64_t src = treloc[r];
    if (src < 0) return;
    const int64_t dst = raw_off[frame_vids[r]];
    const int64_t cnt = int64_t(tbase[r]) * 3;
    for (int64_t e = lane; e < cnt; e += 32) {
        axyz[dst * 3 + e] = axyz[src * 3 + e];
        argb[dst * 3 + e] = argb[src * 3 + e];
    }
}

// append the frame's points in (first-touch rank, frame index) order
__global__ void k_append(const uint32_t* srank, const uint32_t* sidx, int64_t kept,
                         const int32_t* tseg, const int32_t* tbase, const int32_t* frame_vids,
                         const int64_t* raw_off, const double* __restrict__ xyz,
                         const double* __restrict__ rgb, double* axyz, double* argb) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= kept) return;
    const uint32_t r = srank[j];
    const int64_t i = sidx[j];
    const int64_t dst = raw_off[frame_vids[r]] + tbase[r] + (j - tseg[r]);
    axyz[dst * 3 + 0] = xyz[i * 3 + 0];
    axyz[dst * 3 + 1] = xyz[i * 3 + 1];
    axyz[dst * 3 + 2] = xyz[i * 3 + 2];
    argb[dst * 3 + 0] = rgb[i * 3 + 0];
    argb[dst * 3 + 1] = rgb[i * 3 + 1];
    argb[dst * 3 + 2] = rgb[i * 3 + 2];
}

__global__ void k_touched_finish(const int32_t* frame_vids, const int32_t* tbase, const int32_t* tcnt,
                                 int64_t U, int tau, int32_t* raw_count, uint8_t* state, uint8_t* fa,
                                 long long* ctr) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= U) return;
    const int32_t vid = frame_vids[r];
    const int32_t c = tbase[r] + tcnt[r];
    raw_count[vid] = c;
    uint8_t st = state[vid];
    if (st == VX_UNREADY && c >= tau) {       // voxel_map.py:339-340
        st = VX_READY;
        state[vid] = st;
        agg_add(reinterpret_cast<unsigned long long*>(ctr), C_READY);
    }
    fa[r] = st;
}

__global__ void k_rehash(const uint64_t* pkey, int64_t V, uint64_t* tkeys, int32_t* tvals,
                         int64_t tmask) {
    const int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (v >= V) return;
    const uint64_t pk = pkey[v];
    uint64_t h = mix64(pk) & uint64_t(tmask);
    while (true) {
        uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(tkeys + h),
                                  (unsigned long long)EMPTY_KEY, (unsigned long long)pk);
        if (prev == EMPTY_KEY) {
            tvals[h] = int32_t(v);
            return;
        }
        h = (h + 1) & uint64_t(tmask);
    }
}

// ---- densify
__global__ void k_dens_flags(const int32_t* frame_vids, int64_t U, const uint8_t* state,
                             int32_t* cflag) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= U) return;
    const uint8_t st = state[frame_vids[r]];
    cflag[r] = (st == VX_READY || st == VX_ACTIVE) ? 1 : 0;   // gpr.py:283
}

__global__ void k_dens_list(const int32_t* frame_vids, const int32_t* cflag, const int32_t* cscan,
                            int64_t U, const int32_t* raw_count, const uint8_t* has_pred,
                            int32_t* pred_slot, int M, int64_t slot_base, int32_t* cand_voxel,
                            int32_t* cand_n, uint8_t* cand_status, long long* ctr) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= U || !cflag[r]) return;
    const int32_t s = cscan[r];
    const int32_t vid = frame_vids[r];
    const int32_t n = raw_count[vid] + (has_pred[vid] ? M : 0);
    cand_voxel[s] = vid;
    cand_n[s] = n;
    cand_status[s] = 255;
    agg_max(reinterpret_cast<unsigned long long*>(ctr + C_MAXN), unsigned(n));
    if (pred_slot[vid] < 0) {
        const long long k = agg_add(reinterpret_cast<unsigned long long*>(ctr), C_NEWSLOTS);
        pred_slot[vid] = int32_t(slot_base + k);
    }
}

__global__ void k_dens_finish(const uint8_t* status, const uint8_t* before, const uint8_t* after,
                              int64_t S, int32_t* okflag, long long* ctr) {
    const int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const uint8_t st = status[s];
    okflag[s] = st == VX_ST_OK ? 1 : 0;
    unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
    if (st == VX_ST_OK) {
        if (before[s] == VX_READY) agg_add(c, C_FIRST);
        if (after[s] == VX_CONVERGED) agg_add(c, C_CONV);
    } else {
        agg_add(c, st == VX_ST_DEGENERATE ? C_DEGEN : C_CHOL);
    }
}

__global__ void k_compact(const int32_t* flag, const int32_t* scan, const int32_t* vals, int64_t n,
                          int32_t* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) out[scan[i]] = vals[i];
}

__global__ void k_first_solves(const int32_t* cand_voxel, const uint8_t* status, const uint8_t* before,
                               const int32_t* okscan, int64_t S, int32_t* out_flag) {
    const int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= S) return;
    out_flag[s] = (status[s] == VX_ST_OK && before[s] == VX_READY) ? 1 : 0;
}

void map_delete(VxMap* m);

// ------------------------------------------------------------------ helpers
static inline unsigned nblk(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

template <typename T>
static int grow_array(DevBuf& b, int64_t old_n, int64_t new_n, cudaStream_t s) {
    const size_t want = size_t(new_n) * sizeof(T);
    if (b.bytes >= want) return VX_OK;
    void* p = nullptr;
    VX_CUDA(cudaMalloc(&p, want));
    if (b.ptr && old_n > 0) VX_CUDA(cudaMemcpyAsync(p, b.ptr, size_t(old_n) * sizeof(T),
                                                    cudaMemcpyDeviceToDevice, s));
    if (b.ptr) VX_CUDA(cudaFree(b.ptr));   // waits for the copy
    b.ptr = p;
    b.bytes = want;
    return VX_OK;
}

// The counters cross to the host through MAPPED pinned memory, written by a
// one-warp kernel, not by cudaMemcpyAsync: a copy would queue on the copy
// engine behind whatever bulk transfer is in flight (the next frame's H2D, the
// previous frame's record D2H in MappingEngine.ingest_stream), and each of the
// ingest's counter reads would wait for it.
__global__ void k_copy_i64(int64_t* __restrict__ dst, const int64_t* __restrict__ src, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

constexpr int64_t SMALL_FRAME_CANDIDATES = 65536;

static bool ensure_bucket_streams(VxMap* m) {
    if (m->bfork) return true;
    if (m->bstream[0]) return false;      // an earlier attempt failed part-way: stay serial
    for (int b = 0; b < 8; ++b) {
        if (cudaStreamCreateWithFlags(&m->bstream[b], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&m->bdone[b], cudaEventDisableTiming) != cudaSuccess)
            return false;
    }
    if (cudaEventCreateWithFlags(&m->bfork, cudaEventDisableTiming) != cudaSuccess) {
        m->bfork = nullptr;
        return false;
    }
    return true;
}

static int read_counters(VxMap* m, cudaStream_t s) {
    k_copy_i64<<<1, 64, 0, s>>>(m->host_counters_dev, m->counters.as<int64_t>(), C_COUNT);
    count_launch();
    VX_CHECK_LAUNCH();
    VX_CUDA(cudaStreamSynchronize(s));
    return VX_OK;
}

static long long* ctr(VxMap* m) { return m->counters.as<long long>(); }

static int ensure_voxels(VxMap* m, int64_t need, cudaStream_t s) {
    if (need <= m->vcap) return VX_OK;
    int64_t cap = std::max<int64_t>(m->vcap * 2, std::max<int64_t>(need, 1024));
    const int64_t n = m->num_voxels;
    VX_TRY(grow_array<int64_t>(m->keys3, n * 3, cap * 3, s));
    VX_TRY(grow_array<uint64_t>(m->pkey, n, cap, s));
    VX_TRY(grow_array<uint8_t>(m->state, n, cap, s));
    VX_TRY(grow_array<int8_t>(m->axis, n, cap, s));
    VX_TRY(grow_array<int32_t>(m->raw_count, n, cap, s));
    VX_TRY(grow_array<int64_t>(m->raw_off, n, cap, s));
    VX_TRY(grow_array<int32_t>(m->raw_cap, n, cap, s));
    VX_TRY(grow_array<int32_t>(m->pred_slot, n, cap, s));
    VX_TRY(grow_array<uint8_t>(m->has_pred, n, cap, s));
    VX_TRY(grow_array<int32_t>(m->last_first, n, cap, s));
    m->vcap = cap;
    return VX_OK;
}

static int ensure_arena(VxMap* m, int64_t need, cudaStream_t s) {
    if (need <= m->arena_cap) return VX_OK;
    int64_t cap = std::max<int64_t>(m->arena_cap * 2, std::max<int64_t>(need, 1 << 16));
    VX_TRY(grow_array<double>(m->axyz, m->arena_top * 3, cap * 3, s));
    VX_TRY(grow_array<double>(m->argb, m->arena_top * 3, cap * 3, s));
    m->arena_cap = cap;
    return VX_OK;
}

static int ensure_slots(VxMap* m, int64_t need, cudaStream_t s) {
    if (need <= m->slot_cap) return VX_OK;
    int64_t cap = std::max<int64_t>(m->slot_cap * 2, std::max<int64_t>(need, 256));
    const int64_t M = m->M;
    VX_TRY(grow_array<double>(m->pxyz, m->num_slots * M * 3, cap * M * 3, s));
    VX_TRY(grow_array<double>(m->prgb, m->num_slots * M * 3, cap * M * 3, s));
    VX_TRY(grow_array<double>(m->pvar, m->num_slots * M, cap * M, s));
    m->slot_cap = cap;
    return VX_OK;
}

// (re)build the hash table with capacity >= want slots
static int rebuild_table(VxMap* m, int64_t want, cudaStream_t s) {
    int64_t cap = 1024;
    while (cap < want) cap *= 2;
    if (cap != m->tcap) {
        m->tkeys.release();
        m->tvals.release();
        m->tfirst.release();
        m->trank.release();
        VX_TRY(m->tkeys.reserve(cap * 8, s));
        VX_TRY(m->tvals.reserve(cap * 4, s));
        VX_TRY(m->tfirst.reserve(cap * 8, s));
        VX_TRY(m->trank.reserve(cap * 4, s));
        m->tcap = cap;
        k_fill_u64<<<nblk(cap), 256, 0, s>>>(m->tfirst.as<uint64_t>(), cap, ~0ull);
        count_launch();
    }
    k_fill_u64<<<nblk(cap), 256, 0, s>>>(m->tkeys.as<uint64_t>(), cap, EMPTY_KEY);
    count_launch();
    VX_CUDA(cudaMemsetAsync(m->tvals.ptr, 0xff, size_t(cap) * 4, s));
    if (m->num_voxels > 0) {
        k_rehash<<<nblk(m->num_voxels), 256, 0, s>>>(m->pkey.as<uint64_t>(), m->num_voxels,
                                                     m->tkeys.as<uint64_t>(), m->tvals.as<int32_t>(),
                                                     cap - 1);
        count_launch();
    }
    VX_CHECK_LAUNCH();
    return VX_OK;
}

static int bits_for(int64_t v) {
    int b = 0;
    while ((int64_t(1) << b) <= v) ++b;
    return b;
}

// ------------------------------------------------------------------ input slicing (N > 1)
// A rank holding a slice of a scan sends each point to the rank that owns its
// voxel.  Owner = shard_of(key) exactly as k_hash_points computes it; a point
// whose key cannot be formed (non-finite, outside the lattice) goes to rank 0,
// whose hashing kernel then reports it.  Per-CTA owner histograms feed the
// world counters with one atomic per owner and CTA.
__global__ void k_owner_of_points(const double* __restrict__ xyz, int64_t n, double vs, int world,
                                  uint32_t* owner, unsigned long long* counts) {
    __shared__ unsigned int h[65];
    for (int w = threadIdx.x; w <= world; w += blockDim.x) h[w] = 0;
    __syncthreads();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        const double x = xyz[i * 3], y = xyz[i * 3 + 1], z = xyz[i * 3 + 2];
        uint32_t o = 0;
        bool valid = false;
        if (isfinite(x) && isfinite(y) && isfinite(z)) {
            const double fx = floor(xdiv(x, vs)), fy = floor(xdiv(y, vs)), fz = floor(xdiv(z, vs));
            const double lim = double(KEY_LIM);
            if (fx >= -lim && fx < lim && fy >= -lim && fy < lim && fz >= -lim && fz < lim) {
                o = shard_of(pack_key(int64_t(fx), int64_t(fy), int64_t(fz)), world);
                valid = true;
            }
        }
        owner[i] = o;
        atomicAdd(&h[o], 1u);
        if (!valid) atomicAdd(&h[world], 1u);     // counted apart as well
    }
    __syncthreads();
    for (int w = threadIdx.x; w <= world; w += blockDim.x)
        if (h[w]) atomicAdd(counts + w, (unsigned long long)h[w]);
}

// rows of the owner-grouped permutation (stable: frame order within an owner)
__global__ void k_gather_partition(const uint32_t* perm, int64_t n, int64_t gbase,
                                   const double* __restrict__ xyz, const double* __restrict__ rgb,
                                   double* oxyz, double* orgb, int64_t* ogidx) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int64_t i = perm[j];
    oxyz[j * 3] = xyz[i * 3];
    oxyz[j * 3 + 1] = xyz[i * 3 + 1];
    oxyz[j * 3 + 2] = xyz[i * 3 + 2];
    orgb[j * 3] = rgb[i * 3];
    orgb[j * 3 + 1] = rgb[i * 3 + 1];
    orgb[j * 3 + 2] = rgb[i * 3 + 2];
    ogidx[j] = gbase + i;
}

int map_partition_by_owner(VxMap* m, const double* xyz, const double* rgb, int64_t n,
                           int64_t gbase, double* oxyz, double* orgb, int64_t* ogidx,
                           int64_t* h_counts, cudaStream_t s) {
    const int world = m->cfg.shard_world > 1 ? m->cfg.shard_world : 1;
    if (world > 64) {
        set_error("input slicing supports up to 64 shards (got %d)", world);
        return VX_E_INPUT;
    }
    for (int w = 0; w <= world; ++w) h_counts[w] = 0;
    if (n <= 0) return VX_OK;
    if (n >= (int64_t(1) << 31) - 1) {
        set_error("slice of %lld points exceeds the 2^31 point limit", (long long)n);
        return VX_E_INPUT;
    }
    VX_TRY(m->prank.reserve(n * 4, s));
    VX_TRY(m->pidx.reserve(n * 4, s));
    VX_TRY(m->prank2.reserve(n * 4, s));
    VX_TRY(m->pidx2.reserve(n * 4, s));
    VX_TRY(m->stage.reserve(65 * 8, s));
    unsigned long long* dcnt = m->stage.as<unsigned long long>();
    VX_CUDA(cudaMemsetAsync(dcnt, 0, 65 * 8, s));
    k_owner_of_points<<<nblk(n), 256, 0, s>>>(xyz, n, m->cfg.voxel_size, world,
                                              m->prank.as<uint32_t>(), dcnt);
    count_launch();
    VX_CHECK_LAUNCH();
    bool in_alt = false;
    VX_TRY(radix_sort_pairs(m->prank.as<uint32_t>(), m->pidx.as<uint32_t>(), m->prank2.as<uint32_t>(),
                            m->pidx2.as<uint32_t>(), n, bits_for(world - 1), m->sort_tmp, s, &in_alt,
                            /*vals_identity=*/true));
    const uint32_t* perm = in_alt ? m->pidx2.as<uint32_t>() : m->pidx.as<uint32_t>();
    k_gather_partition<<<nblk(n), 256, 0, s>>>(perm, n, gbase, xyz, rgb, oxyz, orgb, ogidx);
    count_launch();
    VX_CHECK_LAUNCH();
    unsigned long long hc[65];
    VX_CUDA(cudaMemcpyAsync(hc, dcnt, size_t(world + 1) * 8, cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaStreamSynchronize(s));
    for (int w = 0; w <= world; ++w) h_counts[w] = int64_t(hc[w]);
    return VX_OK;
}

// ------------------------------------------------------------------ store_frame
static int map_store_frame_impl(VxMap* m, const double* xyz, const double* rgb, int64_t n,
                                VxFrameInfo* info, cudaStream_t s);

int map_store_frame(VxMap* m, const double* xyz, const double* rgb, int64_t n, VxFrameInfo* info,
                    cudaStream_t s) {
    prof_begin(P_HASH, s);
    int rc = map_store_frame_impl(m, xyz, rgb, n, info, s);
    prof_end(P_HASH, s);
    return rc;
}

static int map_store_frame_impl(VxMap* m, const double* xyz, const double* rgb, int64_t n,
                                VxFrameInfo* info, cudaStream_t s) {
    m->frame_index += 1;   // voxel_map.py:320 increments before anything else
    m->frame_touched = 0;
    VxFrameInfo fi{};
    fi.frame_index = m->frame_index;
    fi.points_in = n;
    if (n <= 0) {
        if (info) *info = fi;
        return VX_OK;
    }
    if (n >= (int64_t(1) << 31) - 1) {
        set_error("frame of %lld points exceeds the 2^31 point limit", (long long)n);
        return VX_E_INPUT;
    }
    VX_TRY(m->pslot.reserve(n * 4, s));
    VX_TRY(m->flags.reserve(n * 4, s));
    VX_TRY(m->fscan.reserve(n * 4, s));
    VX_TRY(m->prank.reserve(n * 4, s));
    VX_TRY(m->pidx.reserve(n * 4, s));
    VX_TRY(m->prank2.reserve(n * 4, s));
    VX_TRY(m->pidx2.reserve(n * 4, s));
    // table: keep load <= 1/2 even if every point opens a voxel
    // Table sized for load <= 1/2 with an estimate of the frame's new voxels
    // (points / 8): a small table stays (mostly) L2-resident.  If the frame opens more
    // voxels, the insert kernel flags a long probe and the frame is re-hashed
    // into a 4x table (the retry only re-inserts the existing voxels).
    int64_t want = 2 * (m->num_voxels + std::max<int64_t>(n / 8, 4096));
    if (m->tcap < want) VX_TRY(rebuild_table(m, want, s));

    const double vs = m->cfg.voxel_size;
    for (int attempt = 0;; ++attempt) {
        m->epoch += 1;
        VX_CUDA(cudaMemsetAsync(m->counters.ptr, 0, C_COUNT * sizeof(int64_t), s));
        k_hash_points<<<nblk(n), 256, 0, s>>>(xyz, n, vs, m->tkeys.as<uint64_t>(),
                                              m->tfirst.as<uint64_t>(), m->tcap - 1, m->epoch,
                                              m->cfg.shard_rank, m->cfg.shard_world,
                                              m->pslot.as<int32_t>(), ctr(m));
        count_launch();
        VX_CHECK_LAUNCH();
        k_first_flags<<<nblk(n), 256, 0, s>>>(m->pslot.as<int32_t>(), m->tfirst.as<uint64_t>(), n,
                                              m->flags.as<int32_t>());
        count_launch();
        VX_TRY(scan_exclusive_i32(m->flags.as<int32_t>(), m->fscan.as<int32_t>(), n,
                                  reinterpret_cast<int32_t*>(ctr(m) + C_U), m->scan_tmp, s));
        VX_TRY(read_counters(m, s));   // sync 1: errors, U
        const int64_t err = m->host_counters[C_ERR];
        if (err & 1) {
            set_error("cannot hash non-finite positions");
            return VX_E_INPUT;
        }
        if (err & 2) {
            set_error("voxel key outside the supported lattice |k| < 2^20 (voxel_size %g)", vs);
            return VX_E_RANGE;
        }
        if ((err & 4) && attempt < 6) {
            VX_TRY(rebuild_table(m, m->tcap * 4, s));
            continue;
        }
        if (err & 4) {
            set_error("hash table overflow");
            return VX_E_NOMEM;
        }
        break;
    }
    const int64_t U = int32_t(m->host_counters[C_U] & 0xffffffff);
    fi.touched = U;
    m->frame_touched = U;
    if (U == 0) {
        if (info) *info = fi;
        return VX_OK;
    }
    VX_TRY(m->tslot.reserve(U * 4, s));
    VX_TRY(m->tcnt.reserve(U * 4, s));
    VX_TRY(m->tseg.reserve(U * 4, s));
    VX_TRY(m->tnew.reserve(U * 4, s));
    VX_TRY(m->tnewscan.reserve(U * 4, s));
    VX_TRY(m->tneed.reserve(U * 8, s));
    VX_TRY(m->tneedscan.reserve(U * 8, s));
    VX_TRY(m->tbase.reserve(U * 4, s));
    VX_TRY(m->treloc.reserve(U * 8, s));
    VX_TRY(m->frame_vids.reserve(U * 4, s));
    VX_TRY(m->fb.reserve(U, s));
    VX_TRY(m->fa.reserve(U, s));

    k_rank_slots<<<nblk(n), 256, 0, s>>>(m->pslot.as<int32_t>(), m->flags.as<int32_t>(),
                                         m->fscan.as<int32_t>(), n, m->trank.as<int32_t>(),
                                         m->tslot.as<int32_t>(), m->tcnt.as<int32_t>());
    count_launch();
    // pord (the per-voxel ordinals) lives in pidx2, the placed runs in pidx and
    // the big-run list in prank2; the radix fallback below reuses all four
    uint32_t* pord = m->pidx2.as<uint32_t>();
    k_point_rank<<<nblk(n), 256, 0, s>>>(m->pslot.as<int32_t>(), m->trank.as<int32_t>(), n,
                                         uint32_t(U), m->prank.as<uint32_t>(), pord,
                                         m->tcnt.as<int32_t>());
    count_launch();
    VX_CHECK_LAUNCH();
    VX_TRY(scan_exclusive_i32(m->tcnt.as<int32_t>(), m->tseg.as<int32_t>(), U,
                              reinterpret_cast<int32_t*>(ctr(m) + C_KEPT), m->scan_tmp, s));
    k_touched_prep<<<nblk(U), 256, 0, s>>>(m->tslot.as<int32_t>(), m->tcnt.as<int32_t>(), U,
                                           m->tvals.as<int32_t>(), m->raw_count.as<int32_t>(),
                                           m->raw_cap.as<int32_t>(), m->tnew.as<int32_t>(),
                                           m->tneed.as<int64_t>(), ctr(m) + C_MAXSEG);
    count_launch();
    k_place<<<nblk(n), 256, 0, s>>>(m->prank.as<uint32_t>(), pord, n, uint32_t(U),
                                    m->tseg.as<int32_t>(), m->pidx.as<uint32_t>());
    count_launch();
    VX_CHECK_LAUNCH();
    VX_TRY(scan_exclusive_i32(m->tnew.as<int32_t>(), m->tnewscan.as<int32_t>(), U,
                              reinterpret_cast<int32_t*>(ctr(m) + C_NEW), m->scan_tmp, s));
    VX_TRY(scan_exclusive_i64(m->tneed.as<int64_t>(), m->tneedscan.as<int64_t>(), U,
                              reinterpret_cast<int64_t*>(ctr(m) + C_NEED), m->scan_tmp, s));
    VX_TRY(read_counters(m, s));   // sync 2: new voxels, arena rows
    const int64_t n_new = int32_t(m->host_counters[C_NEW] & 0xffffffff);
    const int64_t need = m->host_counters[C_NEED];
    const int64_t kept = int32_t(m->host_counters[C_KEPT] & 0xffffffff);
    const int64_t maxseg = m->host_counters[C_MAXSEG];
    VX_TRY(ensure_voxels(m, m->num_voxels + n_new, s));
    VX_TRY(ensure_arena(m, m->arena_top + need, s));

    CommitArgs ca{m->tslot.as<int32_t>(), m->tnewscan.as<int32_t>(), m->tnew.as<int32_t>(),
                  m->tneed.as<int64_t>(), m->tneedscan.as<int64_t>(), U, m->num_voxels,
                  m->arena_top, m->tkeys.as<uint64_t>(), m->tvals.as<int32_t>(),
                  m->keys3.as<int64_t>(), m->pkey.as<uint64_t>(), m->state.as<uint8_t>(),
                  m->axis.as<int8_t>(), m->raw_count.as<int32_t>(), m->raw_off.as<int64_t>(),
                  m->raw_cap.as<int32_t>(), m->pred_slot.as<int32_t>(), m->has_pred.as<uint8_t>(),
                  m->frame_vids.as<int32_t>(), m->last_first.as<int32_t>(),
                  m->tfirst.as<uint64_t>(), m->fb.as<uint8_t>(), m->tbase.as<int32_t>(),
                  m->treloc.as<int64_t>()};
    k_touched_commit<<<nblk(U), 256, 0, s>>>(ca);
    count_launch();
    k_relocate<<<nblk(U * 32), 256, 0, s>>>(m->treloc.as<int64_t>(), m->frame_vids.as<int32_t>(),
                                            m->tbase.as<int32_t>(), U, m->raw_off.as<int64_t>(),
                                            m->axyz.as<double>(), m->argb.as<double>());
    count_launch();
    if (kept > 0 && maxseg <= SEG_BIG_MAX) {
        // runs restored to frame order per voxel and appended (warp per run;
        // runs of more than SEG_WARP_MAX points by a CTA each)
        int64_t wb = (U + 7) / 8;
        if (wb > int64_t(sm_count()) * 32) wb = int64_t(sm_count()) * 32;
        k_seg_append_warp<<<unsigned(wb), 256, 0, s>>>(
            m->pidx.as<uint32_t>(), m->tseg.as<int32_t>(), m->tcnt.as<int32_t>(), U,
            m->tbase.as<int32_t>(), m->frame_vids.as<int32_t>(), m->raw_off.as<int64_t>(), xyz, rgb,
            m->axyz.as<double>(), m->argb.as<double>(), m->prank2.as<int32_t>(), ctr(m));
        count_launch();
        if (maxseg > SEG_WARP_MAX) {
            k_seg_append_big<<<unsigned(sm_count() * 2), 1024, 0, s>>>(
                m->pidx.as<uint32_t>(), m->tseg.as<int32_t>(), m->tcnt.as<int32_t>(),
                m->tbase.as<int32_t>(), m->frame_vids.as<int32_t>(), m->raw_off.as<int64_t>(), xyz,
                rgb, m->axyz.as<double>(), m->argb.as<double>(), m->prank2.as<int32_t>(), ctr(m));
            count_launch();
        }
    } else if (kept > 0) {
        // a run longer than SEG_BIG_MAX points: stable LSD radix sort of
        // (rank, index) pairs, then the per-point append
        bool in_alt = false;
        VX_TRY(radix_sort_pairs(m->prank.as<uint32_t>(), m->pidx.as<uint32_t>(),
                                m->prank2.as<uint32_t>(), m->pidx2.as<uint32_t>(), n, bits_for(U),
                                m->sort_tmp, s, &in_alt, /*vals_identity=*/true));
        const uint32_t* srank = in_alt ? m->prank2.as<uint32_t>() : m->prank.as<uint32_t>();
        const uint32_t* sidx = in_alt ? m->pidx2.as<uint32_t>() : m->pidx.as<uint32_t>();
        k_append<<<nblk(kept), 256, 0, s>>>(srank, sidx, kept, m->tseg.as<int32_t>(),
                                            m->tbase.as<int32_t>(), m->frame_vids.as<int32_t>(),
                                            m->raw_off.as<int64_t>(), xyz, rgb, m->axyz.as<double>(),
                                            m->argb.as<double>());
        count_launch();
    }
    k_touched_finish<<<nblk(U), 256, 0, s>>>(m->frame_vids.as<int32_t>(), m->tbase.as<int32_t>(),
                                             m->tcnt.as<int32_t>(), U, m->cfg.tau,
                                             m->raw_count.as<int32_t>(), m->state.as<uint8_t>(),
                                             m->fa.as<uint8_t>(), ctr(m));
    count_launch();
    VX_CHECK_LAUNCH();
    m->num_voxels += n_new;
    m->arena_top += need;
    VX_TRY(read_counters(m, s));   // sync 3: transitions
    fi.new_voxels = n_new;
    fi.points_stored = kept;
    fi.ready_transitions = m->host_counters[C_READY];
    if (info) *info = fi;
    return VX_OK;
}

// ------------------------------------------------------------------ densify
static int map_densify_impl(VxMap* m, VxDensifyInfo* info, cudaStream_t s);

int map_densify(VxMap* m, VxDensifyInfo* info, cudaStream_t s) {
    prof_begin(P_DENSIFY, s);
    int rc = map_densify_impl(m, info, s);
    prof_end(P_DENSIFY, s);
    return rc;
}

static int map_densify_impl(VxMap* m, VxDensifyInfo* info, cudaStream_t s) {
    VxDensifyInfo di{};
    m->solve_candidates = 0;
    m->first_count = 0;
    m->solved = 0;
    const int64_t U = m->frame_touched;
    if (U == 0) {
        if (info) *info = di;
        return VX_OK;
    }
    VX_TRY(m->cflag.reserve(U * 4, s));
    VX_TRY(m->cscan.reserve(U * 4, s));
    VX_CUDA(cudaMemsetAsync(m->counters.ptr, 0, C_COUNT * sizeof(int64_t), s));
    k_dens_flags<<<nblk(U), 256, 0, s>>>(m->frame_vids.as<int32_t>(), U, m->state.as<uint8_t>(),
                                         m->cflag.as<int32_t>());
    count_launch();
    VX_TRY(scan_exclusive_i32(m->cflag.as<int32_t>(), m->cscan.as<int32_t>(), U,
                              reinterpret_cast<int32_t*>(ctr(m) + C_S), m->scan_tmp, s));
    VX_TRY(read_counters(m, s));
    const int64_t S = int32_t(m->host_counters[C_S] & 0xffffffff);
    m->solve_candidates = S;
    di.candidates = S;
    if (S == 0) {
        if (info) *info = di;
        return VX_OK;
    }
    VX_TRY(m->cand_voxel.reserve(S * 4, s));
    VX_TRY(m->cand_n.reserve(S * 4, s));
    VX_TRY(m->cand_status.reserve(S, s));
    VX_TRY(m->cand_before.reserve(S, s));
    VX_TRY(m->cand_after.reserve(S, s));
    VX_TRY(m->items.reserve(S * 4, s));
    VX_TRY(m->okflag.reserve(S * 4, s));
    VX_TRY(m->okscan.reserve(S * 4, s));
    VX_TRY(m->solved_vids.reserve(S * 4, s));
    k_dens_list<<<nblk(U), 256, 0, s>>>(m->frame_vids.as<int32_t>(), m->cflag.as<int32_t>(),
                                        m->cscan.as<int32_t>(), U, m->raw_count.as<int32_t>(),
                                        m->has_pred.as<uint8_t>(), m->pred_slot.as<int32_t>(), m->M,
                                        m->num_slots, m->cand_voxel.as<int32_t>(),
                                        m->cand_n.as<int32_t>(), m->cand_status.as<uint8_t>(), ctr(m));
    count_launch();
    VX_CHECK_LAUNCH();
    VX_TRY(read_counters(m, s));
    const int64_t newslots = m->host_counters[C_NEWSLOTS];
    const int max_n = int(m->host_counters[C_MAXN]);
    di.max_train = max_n;
    VX_TRY(ensure_slots(m, m->num_slots + newslots, s));
    m->num_slots += newslots;
    VX_TRY(m->cand_axis.reserve(S, s));
    VX_TRY(m->cand_meanf.reserve(S * 8, s));

    VoxelSolveArgs a{};
    a.cand_voxel = m->cand_voxel.as<int32_t>();
    a.cand_n = m->cand_n.as<int32_t>();
    a.cand_status = m->cand_status.as<uint8_t>();
    a.cand_before = m->cand_before.as<uint8_t>();
    a.cand_after = m->cand_after.as<uint8_t>();
    a.cand_axis = m->cand_axis.as<int8_t>();
    a.cand_meanf = m->cand_meanf.as<double>();
    a.keys = m->keys3.as<int64_t>();
    a.state = m->state.as<uint8_t>();
    a.value_axis = m->axis.as<int8_t>();
    a.raw_count = m->raw_count.as<int32_t>();
    a.raw_offset = m->raw_off.as<int64_t>();
    a.pred_slot = m->pred_slot.as<int32_t>();
    a.has_pred = m->has_pred.as<uint8_t>();
    a.raw_xyz = m->axyz.as<double>();
    a.raw_rgb = m->argb.as<double>();
    a.pred_xyz = m->pxyz.as<double>();
    a.pred_rgb = m->prgb.as<double>();
    a.pred_var = m->pvar.as<double>();
    a.voxel_size = m->cfg.voxel_size;
    a.sensor_var = m->cfg.sensor_var;
    a.eta = m->cfg.eta;
    a.lam = m->cfg.kernel_lambda;
    a.jitter = m->cfg.jitter;
    a.n_s = m->cfg.n_s;
    a.n_r = m->cfg.n_r;
    a.kernel = m->cfg.kernel;
    a.M = m->M;

    // PCA prepass: value axis, degeneracy, target mean; bucket counts
    prof_begin(P_PCA, s);
    VX_TRY(launch_pca_prepass(a, int(S), ctr(m) + C_B0, s));
    prof_end(P_PCA, s);
    VX_TRY(read_counters(m, s));
    int64_t counts[NUM_BUCKETS], offs[NUM_BUCKETS];
    int64_t acc = 0;
    for (int b = 0; b < NUM_BUCKETS; ++b) {
        counts[b] = m->host_counters[C_B0 + b];
        offs[b] = acc;
        acc += counts[b];
        m->host_counters[C_O0 + b] = offs[b];
    }
    // (host -> device through the mapped counters, off the copy engines)
    k_copy_i64<<<1, 32, 0, s>>>(reinterpret_cast<int64_t*>(ctr(m)) + C_O0, m->host_counters_dev + C_O0,
                                NUM_BUCKETS);
    count_launch();
    VX_TRY(launch_bucket_items(a, int(S), m->items.as<int32_t>(), ctr(m) + C_O0, ctr(m) + C_F0, s));
    // Small frames (one LiDAR scan: a few thousand candidates) are latency-
    // bound per bucket (each launch lasts at least one voxel of its size), so
    // the buckets run concurrently on the map's bucket streams, forked from and
    // joined back into `s`; full-size frames fill the GPU with every bucket and
    // run them back to back, largest first so their tails overlap.
    const bool fork = S <= SMALL_FRAME_CANDIDATES && ensure_bucket_streams(m);
    if (fork) VX_CUDA(cudaEventRecord(m->bfork, s));
    for (int b = NUM_BUCKETS - 1; b >= 0; --b) {
        if (counts[b] == 0) continue;
        a.items = m->items.as<int32_t>() + offs[b];
        a.num_items = int32_t(counts[b]);
        cudaStream_t sb = s;
        if (fork) {
            sb = m->bstream[b];
            VX_CUDA(cudaStreamWaitEvent(sb, m->bfork, 0));
        }
        prof_begin(P_GPR_B0 + b, sb);
        // bucket 7 may take the global-workspace CTA kernel: its own workspace
        VX_TRY(launch_voxel_solve(a, max_n, b == 7 ? m->gpr_work2 : m->gpr_work, sb, b));
        prof_end(P_GPR_B0 + b, sb);
        if (fork) {
            VX_CUDA(cudaEventRecord(m->bdone[b], sb));
            VX_CUDA(cudaStreamWaitEvent(s, m->bdone[b], 0));
        }
    }
    k_dens_finish<<<nblk(S), 256, 0, s>>>(m->cand_status.as<uint8_t>(), m->cand_before.as<uint8_t>(),
                                          m->cand_after.as<uint8_t>(), S, m->okflag.as<int32_t>(),
                                          ctr(m));
    count_launch();
    VX_TRY(scan_exclusive_i32(m->okflag.as<int32_t>(), m->okscan.as<int32_t>(), S,
                              reinterpret_cast<int32_t*>(ctr(m) + C_OK), m->scan_tmp, s));
    k_compact<<<nblk(S), 256, 0, s>>>(m->okflag.as<int32_t>(), m->okscan.as<int32_t>(),
                                      m->cand_voxel.as<int32_t>(), S, m->solved_vids.as<int32_t>());
    count_launch();
    VX_CHECK_LAUNCH();
    VX_TRY(read_counters(m, s));
    di.solved = int32_t(m->host_counters[C_OK] & 0xffffffff);
    di.degenerate = m->host_counters[C_DEGEN];
    di.chol_failed = m->host_counters[C_CHOL];
    di.first_solves = m->host_counters[C_FIRST];
    di.converged = m->host_counters[C_CONV];
    m->solved = di.solved;
    if (info) *info = di;
    return VX_OK;
}

// ------------------------------------------------------------------ ingest
int map_emit_first_gaussians(VxMap* m, const VxCamera* cam, const double* image,
                             const VxSplatConfig* scfg, VxGaussianOut* out, int64_t out_capacity,
                             int64_t* out_records, cudaStream_t s);

int map_ingest(VxMap* m, const double* xyz, const double* rgb, int64_t n, const VxCamera* cam,
               const double* image, const VxSplatConfig* scfg, VxGaussianOut* out,
               int64_t out_capacity, int64_t* out_records, VxFrameInfo* fi, VxDensifyInfo* di,
               cudaStream_t s) {
    VxDensifyInfo dloc{};
    if (out_records) *out_records = 0;
    VX_TRY(map_store_frame(m, xyz, rgb, n, fi, s));
    VX_TRY(map_densify(m, &dloc, s));
    if (di) *di = dloc;
    m->first_count = 0;
    if (cam == nullptr || dloc.first_solves == 0) return VX_OK;
    const int64_t S = m->solve_candidates;
    // first solves in update order: status OK and READY before (pipeline.py:145-156)
    k_first_solves<<<nblk(S), 256, 0, s>>>(m->cand_voxel.as<int32_t>(), m->cand_status.as<uint8_t>(),
                                           m->cand_before.as<uint8_t>(), m->okscan.as<int32_t>(), S,
                                           m->okflag.as<int32_t>());
    count_launch();
    VX_TRY(m->cscan.reserve(S * 4, s));
    VX_TRY(scan_exclusive_i32(m->okflag.as<int32_t>(), m->cscan.as<int32_t>(), S, nullptr,
                              m->scan_tmp, s));
    VX_TRY(m->items.reserve(S * 4, s));
    k_compact<<<nblk(S), 256, 0, s>>>(m->okflag.as<int32_t>(), m->cscan.as<int32_t>(),
                                      m->cand_voxel.as<int32_t>(), S, m->items.as<int32_t>());
    count_launch();
    VX_CHECK_LAUNCH();
    m->first_count = dloc.first_solves;
    if (out == nullptr) {
        // deferred: the first-solve list is kept for vx_map_emit_first_gaussians
        // (the caller stages the image while the frame is solved)
        if (out_records) *out_records = m->first_count * scfg->n_s * scfg->n_s;
        return VX_OK;
    }
    return map_emit_first_gaussians(m, cam, image, scfg, out, out_capacity, out_records, s);
}

// Gaussians of the last ingest's first solves (m->items, update order).  A
// capacity shortfall is reported AFTER the frame has committed, so it must not
// lose the records: *out_records = the required count, VX_E_CAPACITY, and the
// list stays in m->items until the next mutating call, so the caller can grow
// its buffer and call this again (vx_map_emit_first_gaussians).
int map_emit_first_gaussians(VxMap* m, const VxCamera* cam, const double* image,
                             const VxSplatConfig* scfg, VxGaussianOut* out, int64_t out_capacity,
                             int64_t* out_records, cudaStream_t s) {
    if (out_records) *out_records = 0;
    const int64_t cnt = m->first_count;
    if (cnt <= 0 || cam == nullptr || out == nullptr) return VX_OK;
    const int64_t recs = cnt * scfg->n_s * scfg->n_s;
    if (recs > out_capacity) {
        if (out_records) *out_records = recs;
        set_error("Gaussian output capacity %lld < %lld records", (long long)out_capacity,
                  (long long)recs);
        return VX_E_CAPACITY;
    }
    prof_begin(P_SPLAT, s);
    VX_TRY(launch_gaussians(m->pxyz.as<double>(), m->prgb.as<double>(), m->pvar.as<double>(),
                            m->pred_slot.as<int32_t>(), m->items.as<int32_t>(), m->keys3.as<int64_t>(),
                            nullptr, cnt, m->M, *cam, image, *scfg, *out, s));
    prof_end(P_SPLAT, s);
    if (out_records) *out_records = recs;
    return VX_OK;
}

VxMap* map_new(const VxMapConfig& cfg, int* rc) {
    VxMap* m = new (std::nothrow) VxMap();
    if (!m) {
        set_error("out of host memory");
        *rc = VX_E_NOMEM;
        return nullptr;
    }
    m->cfg = cfg;
    m->M = cfg.n_s * cfg.n_r * cfg.n_s * cfg.n_r;
    cudaStream_t s = 0;
    int r = VX_OK;
    if ((r = m->counters.reserve(C_COUNT * sizeof(int64_t), s)) != VX_OK ||
        cudaHostAlloc(&m->host_counters, C_COUNT * sizeof(int64_t), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&m->host_counters_dev), m->host_counters, 0) !=
            cudaSuccess ||
        (r = ensure_voxels(m, std::max<int64_t>(cfg.voxel_capacity, 1024), s)) != VX_OK ||
        (r = ensure_arena(m, std::max<int64_t>(cfg.point_capacity, 1 << 16), s)) != VX_OK ||
        (r = rebuild_table(m, 2 * std::max<int64_t>(cfg.voxel_capacity, 1024), s)) != VX_OK) {
        if (r == VX_OK) {
            set_error("cudaMallocHost failed");
            r = VX_E_NOMEM;
        }
        *rc = r;
        map_delete(m);
        return nullptr;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        set_error("map allocation failed");
        *rc = VX_E_CUDA;
        map_delete(m);
        return nullptr;
    }
    return m;
}

void map_delete(VxMap* m) {
    DevBuf* bufs[] = {&m->tkeys, &m->tvals, &m->tfirst, &m->trank, &m->keys3, &m->pkey, &m->state, &m->last_first,
                      &m->axis, &m->raw_count, &m->raw_off, &m->raw_cap, &m->pred_slot, &m->has_pred,
                      &m->axyz, &m->argb, &m->pxyz, &m->prgb, &m->pvar, &m->pslot, &m->flags,
                      &m->fscan, &m->prank, &m->pidx, &m->prank2, &m->pidx2, &m->tslot, &m->tcnt,
                      &m->tseg, &m->tnew, &m->tnewscan, &m->tneed, &m->tneedscan, &m->tbase,
                      &m->treloc, &m->frame_vids, &m->fb, &m->fa, &m->cflag, &m->cscan,
                      &m->cand_voxel, &m->cand_n, &m->cand_status, &m->cand_before, &m->cand_after,
                      &m->items, &m->okflag, &m->okscan, &m->solved_vids, &m->cand_axis, &m->cand_meanf, &m->counters, &m->scan_tmp,
                      &m->sort_tmp, &m->gpr_work, &m->gpr_work2, &m->stage};
    for (DevBuf* b : bufs) b->release();
    for (int b = 0; b < 8; ++b) {
        if (m->bstream[b]) cudaStreamDestroy(m->bstream[b]);
        if (m->bdone[b]) cudaEventDestroy(m->bdone[b]);
    }
    if (m->bfork) cudaEventDestroy(m->bfork);
    if (m->host_counters) cudaFreeHost(m->host_counters);
    delete m;
}

void map_fill_view(VxMap* m, VxMapView* v) {
    std::memset(v, 0, sizeof(*v));
    v->num_voxels = m->num_voxels;
    v->keys = m->keys3.as<int64_t>();
    v->state = m->state.as<uint8_t>();
    v->value_axis = m->axis.as<int8_t>();
    v->raw_count = m->raw_count.as<int32_t>();
    v->raw_offset = m->raw_off.as<int64_t>();
    v->pred_slot = m->pred_slot.as<int32_t>();
    v->has_pred = m->has_pred.as<uint8_t>();
    v->last_first = m->last_first.as<int32_t>();
    v->raw_xyz = m->axyz.as<double>();
    v->raw_rgb = m->argb.as<double>();
    v->pred_points = m->M;
    v->pred_xyz = m->pxyz.as<double>();
    v->pred_rgb = m->prgb.as<double>();
    v->pred_var = m->pvar.as<double>();
    v->frame_touched = m->frame_touched;
    v->frame_voxels = m->frame_vids.as<int32_t>();
    v->frame_state_before = m->fb.as<uint8_t>();
    v->frame_state_after = m->fa.as<uint8_t>();
    v->solve_candidates = m->solve_candidates;
    v->solve_voxels = m->cand_voxel.as<int32_t>();
    v->solve_status = m->cand_status.as<uint8_t>();
    v->solve_state_before = m->cand_before.as<uint8_t>();
    v->solve_state_after = m->cand_after.as<uint8_t>();
    v->solved = m->solved;
    v->solved_voxels = m->solved_vids.as<int32_t>();
    v->frame_index = m->frame_index;
}

int map_init_gaussians(VxMap* m, const int32_t* vids, int64_t count, const VxCamera& cam,
                       const double* image, const VxSplatConfig& cfg, const VxGaussianOut& out,
                       cudaStream_t s) {
    return launch_gaussians(m->pxyz.as<double>(), m->prgb.as<double>(), m->pvar.as<double>(),
                            m->pred_slot.as<int32_t>(), vids, m->keys3.as<int64_t>(), nullptr, count,
                            m->M, cam, image, cfg, out, s);
}

// ---- key lookup / explicit update sets / host-supplied predictions
__global__ void k_lookup(const int64_t* keys, int64_t n, const uint64_t* tkeys, const int32_t* tvals,
                         int64_t tmask, int32_t* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t a = keys[i * 3], b = keys[i * 3 + 1], c = keys[i * 3 + 2];
    out[i] = -1;
    if (a < -KEY_LIM || a >= KEY_LIM || b < -KEY_LIM || b >= KEY_LIM || c < -KEY_LIM || c >= KEY_LIM)
        return;
    const uint64_t pk = pack_key(a, b, c);
    uint64_t h = mix64(pk) & uint64_t(tmask);
    for (int64_t probe = 0; probe <= tmask; ++probe) {
        const uint64_t cur = tkeys[h];
        if (cur == pk) {
            out[i] = tvals[h];
            return;
        }
        if (cur == EMPTY_KEY) return;
        h = (h + 1) & uint64_t(tmask);
    }
}

int map_lookup(VxMap* m, const int64_t* keys, int64_t n, int32_t* out, cudaStream_t s) {
    if (n <= 0) return VX_OK;
    if (m->tcap == 0) {
        VX_CUDA(cudaMemsetAsync(out, 0xff, size_t(n) * 4, s));
        return VX_OK;
    }
    k_lookup<<<nblk(n), 256, 0, s>>>(keys, n, m->tkeys.as<uint64_t>(), m->tvals.as<int32_t>(),
                                     m->tcap - 1, out);
    count_launch();
    VX_CHECK_LAUNCH();
    return VX_OK;
}

__global__ void k_count_missing(const int32_t* vids, int64_t n, long long* ctr) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && vids[i] < 0) atomicAdd(reinterpret_cast<unsigned long long*>(ctr + C_ERR), 1ull);
}

// Replace the "last frame" voxel list with explicit keys (an update set that
// is not the map's latest frame).  VX_E_CONTRACT if a key is unknown.
int map_set_frame_keys(VxMap* m, const int64_t* keys, int64_t n, cudaStream_t s) {
    VX_TRY(m->frame_vids.reserve(std::max<int64_t>(n, 1) * 4, s));
    VX_TRY(map_lookup(m, keys, n, m->frame_vids.as<int32_t>(), s));
    VX_CUDA(cudaMemsetAsync(m->counters.ptr, 0, C_COUNT * sizeof(int64_t), s));
    if (n > 0) {
        k_count_missing<<<nblk(n), 256, 0, s>>>(m->frame_vids.as<int32_t>(), n, ctr(m));
        count_launch();
    }
    VX_TRY(read_counters(m, s));
    if (m->host_counters[C_ERR] != 0) {
        m->frame_touched = 0;
        set_error("%lld keys of the update set are not in the map", (long long)m->host_counters[C_ERR]);
        return VX_E_CONTRACT;
    }
    m->frame_touched = n;
    return VX_OK;
}

__global__ void k_apply_pred(int32_t vid, const double* xyz, const double* rgb, const double* var, int M,
                             double eta, uint8_t* state, uint8_t* has_pred, const int32_t* pred_slot,
                             double* pxyz, double* prgb, double* pvar, uint8_t* ba) {
    __shared__ double v[256];
    const int slot = pred_slot[vid];
    for (int q = threadIdx.x; q < M; q += blockDim.x) {
        const int64_t pr = int64_t(slot) * M + q;
        for (int d = 0; d < 3; ++d) {
            pxyz[pr * 3 + d] = xyz[q * 3 + d];
            prgb[pr * 3 + d] = rgb[q * 3 + d];
        }
        const double c = var[q] < 0.0 ? 0.0 : var[q];   // np.clip(., 0, None) (voxel_map.py:258)
        pvar[pr] = c;
        v[q] = var[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // classify on the prediction's own (unclipped) mean (voxel_map.py:169-170,237-239)
        const double mean = xdiv(np_pairwise_sum([&](int i) { return v[i]; }, M), double(M));
        ba[0] = state[vid];
        const uint8_t after = mean <= eta ? VX_CONVERGED : VX_ACTIVE;
        state[vid] = after;
        has_pred[vid] = 1;
        ba[1] = after;
    }
}

int map_apply_prediction(VxMap* m, const int64_t* h_key, const double* xyz, const double* rgb,
                         const double* var, int64_t M, uint8_t* h_before_after, cudaStream_t s) {
    if (M != m->M) {
        set_error("prediction has %lld points, the map stores %d per voxel", (long long)M, m->M);
        return VX_E_CONTRACT;
    }
    VX_TRY(m->stage.reserve(256, s));
    int64_t* dkey = m->stage.as<int64_t>();
    int32_t* dvid = reinterpret_cast<int32_t*>(dkey + 4);
    uint8_t* dba = reinterpret_cast<uint8_t*>(dkey + 6);
    VX_CUDA(cudaMemcpyAsync(dkey, h_key, 3 * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    VX_TRY(map_lookup(m, dkey, 1, dvid, s));
    int32_t vid = -1;
    uint8_t st = 0;
    int32_t slot = -1;
    VX_CUDA(cudaMemcpyAsync(&vid, dvid, 4, cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaStreamSynchronize(s));
    if (vid < 0) {
        set_error("voxel (%lld, %lld, %lld) is not in the map", (long long)h_key[0],
                  (long long)h_key[1], (long long)h_key[2]);
        return VX_E_INPUT;   // KeyError in the binding
    }
    VX_CUDA(cudaMemcpyAsync(&st, m->state.as<uint8_t>() + vid, 1, cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaMemcpyAsync(&slot, m->pred_slot.as<int32_t>() + vid, 4, cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaStreamSynchronize(s));
    if (st != VX_READY && st != VX_ACTIVE) {
        static const char* names[4] = {"UNREADY", "READY", "ACTIVE", "CONVERGED"};
        set_error("cell (%lld, %lld, %lld) in state %s cannot accept a solve", (long long)h_key[0],
                  (long long)h_key[1], (long long)h_key[2], names[st & 3]);
        return VX_E_CONTRACT;
    }
    if (slot < 0) {
        VX_TRY(ensure_slots(m, m->num_slots + 1, s));
        slot = int32_t(m->num_slots++);
        VX_CUDA(cudaMemcpyAsync(m->pred_slot.as<int32_t>() + vid, &slot, 4, cudaMemcpyHostToDevice, s));
    }
    if (M > 256) {
        set_error("prediction larger than 256 points");
        return VX_E_CONTRACT;
    }
    k_apply_pred<<<1, 256, 0, s>>>(vid, xyz, rgb, var, int(M), m->cfg.eta, m->state.as<uint8_t>(),
                                   m->has_pred.as<uint8_t>(), m->pred_slot.as<int32_t>(),
                                   m->pxyz.as<double>(), m->prgb.as<double>(), m->pvar.as<double>(), dba);
    count_launch();
    VX_CHECK_LAUNCH();
    VX_CUDA(cudaMemcpyAsync(h_before_after, dba, 2, cudaMemcpyDeviceToHost, s));
    VX_CUDA(cudaStreamSynchronize(s));
    return VX_OK;
}

int map_configure_solver(VxMap* m, int n_s, int n_r, double lam, double jitter, int kernel) {
    const int M = n_s * n_r * n_s * n_r;
    if (n_s < 1 || n_r < 1 || n_s * n_r > 16) {
        set_error("n_s, n_r must be >= 1 with n_s * n_r <= 16");
        return VX_E_INPUT;
    }
    if (!(lam > 0)) {
        set_error("kernel constant must be positive");
        return VX_E_INPUT;
    }
    if (M != m->M && m->num_slots > 0) {
        set_error("the map already holds %d-point predictions; cannot switch to %d", m->M, M);
        return VX_E_CONTRACT;
    }
    m->M = M;
    m->cfg.n_s = n_s;
    m->cfg.n_r = n_r;
    m->cfg.kernel_lambda = lam;
    m->cfg.jitter = jitter;
    m->cfg.kernel = kernel;
    return VX_OK;
}

int map_clear(VxMap* m, cudaStream_t s) {
    m->num_voxels = 0;
    m->arena_top = 0;
    m->num_slots = 0;
    m->frame_touched = 0;
    m->solve_candidates = 0;
    m->first_count = 0;
    m->solved = 0;
    m->frame_index = -1;
    if (m->tcap > 0) {
        k_fill_u64<<<nblk(m->tcap), 256, 0, s>>>(m->tkeys.as<uint64_t>(), m->tcap, EMPTY_KEY);
        count_launch();
        VX_CUDA(cudaMemsetAsync(m->tvals.ptr, 0xff, size_t(m->tcap) * 4, s));
        VX_CHECK_LAUNCH();
    }
    return VX_OK;
}

}  // namespace vx
