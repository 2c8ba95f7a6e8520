// Micro-benchmark: issue rates of the instruction forms used by the hot loops
// (FFMA, FFMA2, FADD2, FFMA.SAT, FMNMX, LEA/IMAD, LDS, LDS.64) on this GPU.
// Prints warp-instructions per clock per SM for each form.
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 512

template <int KIND>
__global__ void __launch_bounds__(1024, 1) bench(float* out, long long* cyc, int n)
{
    __shared__ float sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = (float)i * 1e-3f;
    __syncthreads();
    float a[CHAINS];
    unsigned long long p[CHAINS];
    unsigned u[CHAINS];
    float q[CHAINS];
    for (int c = 0; c < CHAINS; ++c) {
        a[c] = threadIdx.x * 1e-3f + c;
        q[c] = a[c] - 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(p[c]) : "f"(a[c]), "f"(a[c] + 1.f));
        u[c] = (threadIdx.x * 4 + c * 128) & 0x3ffc;
    }
    const float m = 0.999f, b = 1e-4f;
    unsigned long long m2, b2;
    asm("mov.b64 %0, {%1, %2};" : "=l"(m2) : "f"(m), "f"(m));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b2) : "f"(b), "f"(b));
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (KIND == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(m), "f"(b));
            if (KIND == 1) asm volatile("fma.rn.f32 %0, %0, %1, 0f38D1B717;" : "+f"(a[c]) : "f"(m));
            if (KIND == 2) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(m2), "l"(b2));
            if (KIND == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(b2));
            if (KIND == 4) asm volatile("fma.rn.sat.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(m), "f"(b));
            if (KIND == 5) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(b));
            if (KIND == 6) asm volatile("mad.lo.u32 %0, %0, 4, %1;" : "+r"(u[c]) : "r"(sbase));
            if (KIND == 7) {
                float v;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(sbase + (u[c] & 0x3ffc)));
                u[c] += __float_as_uint(v) & 4;
            }
            if (KIND == 8) {
                float v, w;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v), "=f"(w) : "r"(sbase + (u[c] & 0x3ff8)));
                u[c] += (__float_as_uint(v) ^ __float_as_uint(w)) & 8;
            }
            if (KIND == 9) {  // FFMA2 + FMNMX mix (co-issue across pipes)
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(m2), "l"(b2));
                asm volatile("max.f32 %0, %0, %1;" : "+f"(q[c]) : "f"(b));
            }
            if (KIND == 10) {  // FFMA + FMNMX
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(m), "f"(b));
                asm volatile("max.f32 %0, %0, %1;" : "+f"(q[c]) : "f"(b));
            }
            if (KIND == 11) asm volatile("add.rm.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(b2));
            if (KIND == 13) {  // LDS.128
                float v, w, x, y;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v), "=f"(w), "=f"(x), "=f"(y) : "r"(sbase + (u[c] & 0x3ff0)));
                u[c] += (__float_as_uint(v) ^ __float_as_uint(w) ^ __float_as_uint(x) ^ __float_as_uint(y)) & 16;
            }
            if (KIND == 14) {  // LDS.32, lanes spread over 45 words (forward-like: 2 wavefronts some of the time)
                float v;
                const unsigned l = threadIdx.x & 31;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(sbase + (((u[c] & 0x3f00) + ((l * 45) / 32) * 4))));
                u[c] += __float_as_uint(v) & 4;
            }
            if (KIND == 15) {  // LDS.64, lanes spread over 45 words (8B elements)
                float v, w;
                const unsigned l = threadIdx.x & 31;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v), "=f"(w) : "r"(sbase + (((u[c] & 0x3e00) + ((l * 45) / 32) * 8))));
                u[c] += (__float_as_uint(v) ^ __float_as_uint(w)) & 8;
            }
            if (KIND == 16) {  // FFMA2 + FFMA: pipe sharing
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(m2), "l"(b2));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(m), "f"(b));
            }
            if (KIND == 17) {  // 2 x LDS.32 of adjacent words (pair taps) + 2 alu
                float v, w;
                asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+4];" : "=f"(v), "=f"(w) : "r"(sbase + (u[c] & 0x3ff8)));
                u[c] += (__float_as_uint(v) ^ __float_as_uint(w)) & 8;
            }
            if (KIND == 18) {  // IMAD x,4,y explicit and LEA
                asm volatile("{.reg .u32 t; shl.b32 t, %0, 2; add.u32 %0, t, %1;}" : "+r"(u[c]) : "r"(sbase));
            }
            if (KIND == 12) asm volatile("shl.b32 %0, %0, 2;\n\tadd.u32 %0, %0, %1;" : "+r"(u[c]) : "r"(sbase));
        }
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int c = 0; c < CHAINS; ++c) {
        float x, y;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(p[c]));
        s += a[c] + x + y + (float)u[c] + q[c];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(const char* name, int per_chain_instr)
{
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    cudaMalloc(&cyc, 148 * sizeof(long long));
    bench<K><<<148, 1024>>>(out, cyc, 16);
    bench<K><<<148, 1024>>>(out, cyc, ITERS);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double warp_instr = 32.0 * ITERS * CHAINS * per_chain_instr;  // per SM (32 warps)
    printf("%-22s %.3f warp-instr/clk/SM  (%.3f per SMSP)\n", name, warp_instr / c, warp_instr / c / 4);
    cudaFree(out);
    cudaFree(cyc);
}

int main()
{
    run<0>("FFMA reg", 1);
    run<1>("FFMA imm", 1);
    run<2>("FFMA2", 1);
    run<3>("FADD2", 1);
    run<11>("FADD2.RM", 1);
    run<4>("FFMA.SAT", 1);
    run<5>("FMNMX", 1);
    run<6>("IMAD/LEA", 1);
    run<12>("SHL+IADD", 2);
    run<7>("LDS (+2 alu)", 1);
    run<8>("LDS.64 (+2 alu)", 1);
    run<9>("FFMA2+FMNMX", 2);
    run<13>("LDS.128 (+2 alu)", 1);
    run<14>("LDS span45 (+2alu)", 1);
    run<15>("LDS.64 span45", 1);
    run<16>("FFMA2+FFMA", 2);
    run<17>("2xLDS adj (+2alu)", 2);
    run<18>("SHL+ADD asm", 1);
    run<10>("FFMA+FMNMX", 2);
    return 0;
}
