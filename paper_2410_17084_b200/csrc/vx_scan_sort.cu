// Device-wide exclusive scan and stable LSD radix sort (hand-written; used by
// the hashing stage to reproduce the reference's first-touch order and
// frame-order point grouping, voxel_map.py:324-341).
#include "vx_common.cuh"
#include "vx_internal.h"

namespace vx {

// ------------------------------------------------------------------ scan
constexpr int SCAN_T = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_T * SCAN_ITEMS;

template <typename T>
__device__ T block_exclusive_scan(T v, T* sh, T* total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        T s = lane < SCAN_T / 32 ? sh[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(FULL, s, o);
            if (lane >= o) s += y;
        }
        if (lane < SCAN_T / 32) sh[lane] = s;
    }
    __syncthreads();
    T warp_off = w > 0 ? sh[w - 1] : T(0);
    if (total) *total = sh[SCAN_T / 32 - 1];
    __syncthreads();
    return warp_off + x - v;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_T) scan_tiles(const T* in, T* out, int64_t n, T* tile_sums) {
    __shared__ T sh[32];
    const int64_t base = int64_t(blockIdx.x) * SCAN_TILE + int64_t(threadIdx.x) * SCAN_ITEMS;
    T v[SCAN_ITEMS];
    T run = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        v[k] = (base + k < n) ? in[base + k] : T(0);
        run += v[k];
    }
    T tot;
    T ex = block_exclusive_scan<T>(run, sh, &tot);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        if (base + k < n) out[base + k] = ex;
        ex += v[k];
    }
    if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = tot;
}

template <typename T>
__global__ void scan_add(T* out, int64_t n, const T* tile_off) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] += tile_off[i / SCAN_TILE];
}

template <typename T>
__global__ void scan_total(const T* in, const T* out, int64_t n, T* total) {
    if (n > 0) *total = out[n - 1] + in[n - 1];
    else *total = T(0);
}

template <typename T>
static int scan_exclusive(const T* in, T* out, int64_t n, T* total, DevBuf& tmp, cudaStream_t s,
                          size_t tmp_off) {
    if (n <= 0) {
        if (total) {
            VX_CUDA(cudaMemsetAsync(total, 0, sizeof(T), s));
        }
        return VX_OK;
    }
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles == 1) {
        scan_tiles<T><<<1, SCAN_T, 0, s>>>(in, out, n, nullptr);
        count_launch();
        VX_CHECK_LAUNCH();
    } else {
        // recursion on tile sums; layout in tmp: [sums | sums_scan | deeper...]
        const size_t need = tmp_off + size_t(tiles) * 2 * sizeof(T);
        if (tmp.bytes < need) {
            set_error("scan scratch too small");
            return VX_E_NOMEM;
        }
        T* sums = reinterpret_cast<T*>(static_cast<char*>(tmp.ptr) + tmp_off);
        T* sums_ex = sums + tiles;
        scan_tiles<T><<<unsigned(tiles), SCAN_T, 0, s>>>(in, out, n, sums);
        count_launch();
        VX_CHECK_LAUNCH();
        VX_TRY(scan_exclusive<T>(sums, sums_ex, tiles, nullptr, tmp, s,
                                 tmp_off + size_t(tiles) * 2 * sizeof(T)));
        scan_add<T><<<unsigned((n + 255) / 256), 256, 0, s>>>(out, n, sums_ex);
        count_launch();
        VX_CHECK_LAUNCH();
    }
    if (total) {
        scan_total<T><<<1, 1, 0, s>>>(in, out, n, total);
        count_launch();
        VX_CHECK_LAUNCH();
    }
    return VX_OK;
}

static size_t scan_scratch_bytes(int64_t n, size_t elem) {
    size_t b = 0;
    while (n > SCAN_TILE) {
        int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
        b += size_t(tiles) * 2 * elem;
        n = tiles;
    }
    return b + 256;
}

int scan_exclusive_i32(const int32_t* in, int32_t* out, int64_t n, int32_t* total, DevBuf& tmp,
                       cudaStream_t s) {
    VX_TRY(tmp.reserve(scan_scratch_bytes(n, 4), s));
    return scan_exclusive<int32_t>(in, out, n, total, tmp, s, 0);
}
int scan_exclusive_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total, DevBuf& tmp,
                       cudaStream_t s) {
    VX_TRY(tmp.reserve(scan_scratch_bytes(n, 8), s));
    return scan_exclusive<int64_t>(in, out, n, total, tmp, s, 0);
}

// ------------------------------------------------------------------ radix sort
// Classic three-phase stable LSD pass: per-tile digit histograms (digit-major
// layout), an exclusive scan of that table, and a stable per-tile scatter that
// ranks equal digits by (round, warp, lane) with __match_any_sync.
constexpr int RS_T = 256;
constexpr int RS_ROUNDS = 16;
constexpr int RS_TILE = RS_T * RS_ROUNDS;   // 4096 keys per tile

__global__ void __launch_bounds__(RS_T) rs_hist(const uint32_t* keys, int64_t n, int shift,
                                                int radix, int64_t tiles, int32_t* hist) {
    __shared__ int32_t h[256];
    for (int d = threadIdx.x; d < radix; d += RS_T) h[d] = 0;
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * RS_TILE;
    const uint32_t mask = uint32_t(radix - 1);
    for (int k = 0; k < RS_ROUNDS; ++k) {
        const int64_t i = base + int64_t(k) * RS_T + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & mask], 1);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += RS_T) hist[int64_t(d) * tiles + blockIdx.x] = h[d];
}

// Stable scatter of one tile: keys are ranked in (round, warp, lane) order
// into a shared-memory copy of the tile grouped by digit, which is then
// written out run by run (consecutive threads -> consecutive addresses of a
// digit's run) instead of 2-element fragments per digit per round.
__global__ void __launch_bounds__(RS_T) rs_scatter(const uint32_t* keys, const uint32_t* vals,
                                                   uint32_t* okeys, uint32_t* ovals, int64_t n,
                                                   int shift, int radix, int64_t tiles,
                                                   const int32_t* offs, const int32_t* hist) {
    __shared__ uint32_t sk[RS_TILE];
    __shared__ uint32_t sv[RS_TILE];
    __shared__ int32_t run[256];
    __shared__ int32_t gdelta[256];
    __shared__ int32_t wcnt[RS_T / 32][256];
    __shared__ int32_t wsum[RS_T / 32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // local exclusive scan of this tile's digit counts (radix <= 256 = RS_T)
    const int32_t c = threadIdx.x < radix ? hist[int64_t(threadIdx.x) * tiles + blockIdx.x] : 0;
    int32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    for (int ww = 0; ww < RS_T / 32; ++ww) wcnt[ww][threadIdx.x] = 0;
    __syncthreads();
    int32_t woff = 0;
    for (int ww = 0; ww < w; ++ww) woff += wsum[ww];
    if (threadIdx.x < radix) {
        const int32_t ls = woff + x - c;
        run[threadIdx.x] = ls;
        gdelta[threadIdx.x] = offs[int64_t(threadIdx.x) * tiles + blockIdx.x] - ls;
    }
    __syncthreads();
    const int64_t base = int64_t(blockIdx.x) * RS_TILE;
    const int tn = int(n - base < RS_TILE ? n - base : RS_TILE);
    const uint32_t mask = uint32_t(radix - 1);
    for (int k = 0; k < RS_ROUNDS; ++k) {
        const int li = k * RS_T + threadIdx.x;
        const bool valid = li < tn;
        const uint32_t key = valid ? keys[base + li] : 0u;
        const uint32_t val = valid ? (vals ? vals[base + li] : uint32_t(base + li)) : 0u;   // null: identity
        const int d = valid ? int((key >> shift) & mask) : 256 + lane;   // unique dummy digits
        const unsigned peers = __match_any_sync(FULL, d);
        const int lrank = __popc(peers & lanemask_lt());
        if (valid && lrank == 0) wcnt[w][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int off = run[d] + lrank;
            for (int ww = 0; ww < w; ++ww) off += wcnt[ww][d];
            sk[off] = key;
            sv[off] = val;
        }
        __syncthreads();
        if (threadIdx.x < radix) {
            int tot = 0;
#pragma unroll
            for (int ww = 0; ww < RS_T / 32; ++ww) {
                tot += wcnt[ww][threadIdx.x];
                wcnt[ww][threadIdx.x] = 0;
            }
            run[threadIdx.x] += tot;
        }
        __syncthreads();
    }
    for (int j = threadIdx.x; j < tn; j += RS_T) {
        const uint32_t key = sk[j];
        const int64_t g = int64_t(gdelta[(key >> shift) & mask]) + j;
        okeys[g] = key;
        ovals[g] = sv[j];
    }
}

__global__ void rs_iota(uint32_t* v, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = uint32_t(i);
}

// vals_identity: the values are 0..n-1 and `vals` is only written (the first
// pass generates them instead of reading an iota array)
int radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt,
                     int64_t n, int bits, DevBuf& tmp, cudaStream_t s, bool* result_in_alt,
                     bool vals_identity) {
    *result_in_alt = false;
    if (n <= 1 || bits <= 0) {
        if (vals_identity && n > 0) {
            rs_iota<<<unsigned((n + 255) / 256), 256, 0, s>>>(vals, n);
            count_launch();
            VX_CHECK_LAUNCH();
        }
        return VX_OK;
    }
    const int passes = (bits + 7) / 8;
    const int dbits = (bits + passes - 1) / passes;
    const int radix = 1 << dbits;
    const int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
    const int64_t hn = int64_t(radix) * tiles;
    const size_t hist_bytes = size_t(hn) * 2 * sizeof(int32_t) + 256;
    const size_t need = hist_bytes + scan_scratch_bytes(hn, 4);
    VX_TRY(tmp.reserve(need, s));
    int32_t* hist = tmp.as<int32_t>();
    int32_t* offs = hist + hn;
    uint32_t *ik = keys, *iv = vals, *ok = keys_alt, *ov = vals_alt;
    for (int p = 0; p < passes; ++p) {
        const int shift = p * dbits;
        rs_hist<<<unsigned(tiles), RS_T, 0, s>>>(ik, n, shift, radix, tiles, hist);
        count_launch();
        VX_CHECK_LAUNCH();
        VX_TRY(scan_exclusive<int32_t>(hist, offs, hn, nullptr, tmp, s,
                                       (hist_bytes + 255) & ~size_t(255)));
        rs_scatter<<<unsigned(tiles), RS_T, 0, s>>>(ik, (p == 0 && vals_identity) ? nullptr : iv, ok, ov,
                                                    n, shift, radix, tiles, offs, hist);
        count_launch();
        VX_CHECK_LAUNCH();
        uint32_t* t;
        t = ik; ik = ok; ok = t;
        t = iv; iv = ov; ov = t;
        *result_in_alt = !*result_in_alt;
    }
    return VX_OK;
}
}  // namespace vx
