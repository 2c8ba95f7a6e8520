// Micro-benchmark: shared-memory load throughput (LDS / LDS.64 / LDS.128, conflict-free and
// with the forward projector's 32-rays-over-45-lanes spread), addresses independent of the
// loaded data (throughput, not latency).
#include <cstdio>
#include <cuda_runtime.h>
#define CHAINS 8
#define ITERS 1024
template <int KIND>
__global__ void __launch_bounds__(512, 2) bench(float* out, long long* cyc, int n)
{
    __shared__ __align__(16) float sm[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (float)i * 1e-3f;
    __syncthreads();
    const unsigned l = threadIdx.x & 31;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    float acc[CHAINS];
    unsigned off[CHAINS];
    for (int c = 0; c < CHAINS; ++c) {
        acc[c] = 0.f;
        unsigned e;
        if (KIND == 0) e = l * 4;                       // LDS.32 conflict-free
        if (KIND == 1) e = ((l * 45) / 32) * 4;         // LDS.32 span 45 words
        if (KIND == 2) e = l * 8;                       // LDS.64 conflict-free
        if (KIND == 3) e = ((l * 45) / 32) * 8;         // LDS.64 span 45 elements
        if (KIND == 4) e = l * 16;                      // LDS.128
        if (KIND == 5) e = ((l * 45) / 32) * 4;         // 2 x LDS.32 adjacent, span 45
        if (KIND == 6) e = ((l * 33) / 32) * 4;         // LDS.32 span 33 (gather-like)
        if (KIND == 7) e = ((l * 33) / 32) * 8;         // LDS.64 span 33 (gather pairs)
        off[c] = e + c * 1024 + (threadIdx.x >> 5) * 64;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
        const unsigned sh = (it & 7) * 2048;
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            const unsigned a = sbase + ((off[c] + sh) & 0x7ff0) + (off[c] & 0xf);
            if (KIND == 0 || KIND == 1 || KIND == 6) {
                float v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
                acc[c] += v;
            } else if (KIND == 2 || KIND == 3 || KIND == 7) {
                float v, w;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v), "=f"(w) : "r"(a));
                acc[c] += v * w;
            } else if (KIND == 4) {
                float v, w, x, y;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v), "=f"(w), "=f"(x), "=f"(y) : "r"(a));
                acc[c] += (v + w) * (x + y);
            } else {
                float v, w;
                asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+4];" : "=f"(v), "=f"(w) : "r"(a));
                acc[c] += v * w;
            }
        }
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int c = 0; c < CHAINS; ++c) s += acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int K>
void run(const char* name, int lds_per)
{
    float* out; long long* cyc;
    cudaMalloc(&out, 296 * 512 * sizeof(float));
    cudaMalloc(&cyc, 296 * sizeof(long long));
    bench<K><<<296, 512>>>(out, cyc, 16);
    bench<K><<<296, 512>>>(out, cyc, ITERS);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double wi = 2 * 16.0 * ITERS * CHAINS * lds_per;  // per SM: 2 CTAs x 16 warps
    printf("%-26s %.3f LDS-instr/clk/SM\n", name, wi / c);
}
int main()
{
    run<0>("LDS.32 conflict-free", 1);
    run<1>("LDS.32 span45", 1);
    run<6>("LDS.32 span33", 1);
    run<5>("2xLDS.32 adj span45", 2);
    run<2>("LDS.64 conflict-free", 1);
    run<3>("LDS.64 span45", 1);
    run<7>("LDS.64 span33", 1);
    run<4>("LDS.128 conflict-free", 1);
    return 0;
}
