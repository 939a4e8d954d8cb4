// FP64 tensor-core (m8n8k4 DMMA) and DFMA throughput microbenchmark (B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dmma_peak.cu -o /tmp/dmma_peak && /tmp/dmma_peak
#include <cstdio>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters) {
    double c[CH][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma(double* out, int iters) {
    double c[CH];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) c[i] = fma(a, c[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half the warps issue DMMA chains, the other half DFMA chains: do the two
// FP64 pipes add up?
__global__ void k_mixed(double* out, int iters) {
    const int w = threadIdx.x >> 5;
    double s = 0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    if (w & 1) {
        double c[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    } else {
        double c[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = i;
        for (int it = 0; it < 16 * iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) c[i] = fma(a, c[i], b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += c[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
float time_it(K kern, int blocks, int threads, double* out, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, size_t(sms) * 64 * 1024 * 8);
    const int iters = 4096;
    for (int wps : {1, 2, 4, 8, 16}) {
        const int blocks = sms, threads = 32 * wps;
        float ms = time_it(k_dmma<8>, blocks, threads, out, iters);
        double flops = double(blocks) * wps * iters * 8 * 512.0;   // 8x8x4 x2 flops per mma
        printf("DMMA  %2d warps/SM x 8 chains: %7.2f TFLOP/s  (%.2f cycles/mma/SM at 1.965 GHz)\n", wps,
               flops / ms / 1e9, (ms * 1e-3 * 1.965e9) / (double(wps) * iters * 8));
        ms = time_it(k_dmma<1>, blocks, threads, out, iters);
        flops = double(blocks) * wps * iters * 1 * 512.0;
        printf("DMMA  %2d warps/SM x 1 chain : %7.2f TFLOP/s  (latency %.1f cycles if 1 warp)\n", wps,
               flops / ms / 1e9, (ms * 1e-3 * 1.965e9) / iters);
    }
    for (int wps : {4, 8, 16, 32}) {
        float ms = time_it(k_dfma<8>, sms, 32 * wps, out, iters);
        double flops = double(sms) * 32 * wps * iters * 8 * 2.0;
        printf("DFMA  %2d warps/SM x 8 chains: %7.2f TFLOP/s\n", wps, flops / ms / 1e9);
    }
    for (int wps : {8, 16}) {
        float ms = time_it(k_mixed, sms, 32 * wps, out, iters / 4);
        // wps/2 DMMA warps x 8 chains x 512 flops, wps/2 DFMA warps x 16 x 8 chains x 64 flops
        double fl_dmma = double(sms) * (wps / 2) * (iters / 4) * 8 * 512.0;
        double fl_dfma = double(sms) * (wps / 2) * (iters / 4) * 16 * 8 * 64.0;
        printf("MIXED %2d warps/SM: %7.2f TFLOP/s total (DMMA share %.2f)\n", wps,
               (fl_dmma + fl_dfma) / ms / 1e9, fl_dmma / (fl_dmma + fl_dfma));
    }
    return 0;
}

// dependent-chain latencies (one warp), cycles per operation
__global__ void k_lat(double* out, long long* cyc, int iters) {
    double x = 1.0 + threadIdx.x * 1e-12, y = 0.999999;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-9);
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) x = rsqrt(x) + 0.5;
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) x = __dmul_rn(x, y);
    long long t3 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / iters;
        cyc[1] = (t2 - t1) / iters;
        cyc[2] = (t3 - t2) / iters;
    }
}

__global__ void k_shfl_lat(double* out, long long* cyc, int iters) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
}

__global__ void k_lds_lat(double* out, long long* cyc, int iters) {
    __shared__ int buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) p = buf[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
}

int lat_main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 4096);
    cudaMallocManaged(&cyc, 64);
    k_lat<<<1, 32>>>(out, cyc, 4096);
    k_shfl_lat<<<1, 32>>>(out, cyc, 4096);
    k_lds_lat<<<1, 32>>>(out, cyc, 4096);
    cudaDeviceSynchronize();
    printf("latency (cycles): DFMA %lld, rsqrt(double)+add %lld, DMUL %lld, SHFL+DADD %lld, LDS.32 %lld\n",
           cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
    return 0;
}
static int dummy = lat_main();
