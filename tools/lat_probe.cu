// Latency microbenchmark (one warp, dependent chains, clock64): DFMA, DMUL,
// FP64 rsqrt()/sqrt()/division/exp(), MUFU.RSQ64H (rsqrt approx), m8n8k4 DMMA,
// shfl, LDS, __syncwarp.  Guides the chain design of the GPR kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/lat_probe.cu && /tmp/lat
#include <cstdio>
#include <cuda_runtime.h>

#define N 256
__device__ double sink;

__global__ void k(double seed, long long* out) {
    __shared__ double sm[64];
    const int lane = threadIdx.x;
    sm[lane] = seed + lane;
    sm[lane + 32] = seed;
    __syncwarp();
    double x = seed + lane * 1e-3, y = 1.0000001;
    long long t0, t1;
    int i = 0;
#define TIME(idx, body)                        \
    t0 = clock64();                            \
    for (i = 0; i < N; ++i) { body; }          \
    t1 = clock64();                            \
    if (lane == 0) out[idx] = (t1 - t0);
    TIME(0, x = fma(x, y, 1e-9));
    TIME(1, x = x * y);
    TIME(2, x = rsqrt(x) + 0.5);
    TIME(3, x = sqrt(x) + 0.5);
    TIME(4, x = 1.0 / x + 0.5);
    TIME(5, x = exp(-x) + 0.5);
    double c0 = x, c1 = 0.0;
    TIME(6, asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c0), "+d"(c1) : "d"(y), "d"(y)));
    x += c0 + c1;
    TIME(7, x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31));
    int idx = lane;
    TIME(8, idx = int(sm[idx & 63]) & 63);
    TIME(9, __syncwarp(); x = x * y);
    double r;
    TIME(10, asm volatile("{.reg .f64 t; rsqrt.approx.ftz.f64 t, %1; add.f64 %0, t, 0.5;}" : "=d"(r) : "d"(x)); x = r);
    TIME(11, x = __drcp_rn(x) + 0.5);
    TIME(12, asm volatile("{.reg .f64 t; rcp.approx.ftz.f64 t, %1; add.f64 %0, t, 0.5;}" : "=d"(r) : "d"(x)); x = r);
    sink = x + idx;
}

int main() {
    long long* d;
    long long h[16] = {};
    cudaMalloc(&d, sizeof(h));
    for (int rep = 0; rep < 2; ++rep) k<<<1, 32>>>(1.5, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[] = {"dfma", "dmul", "rsqrt()", "sqrt()", "1/x", "exp()", "dmma m8n8k4",
                           "shfl", "lds", "syncwarp+dmul", "rsqrt.approx.f64", "__drcp_rn", "rcp.approx.f64"};
    for (int i = 0; i < 13; ++i) printf("%-18s %6.1f cycles\n", names[i], double(h[i]) / N);
    return 0;
}
