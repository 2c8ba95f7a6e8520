#include <cstdio>
#include <cuda_runtime.h>
// streaming reference: 7 reads + 3 writes per voxel in the FGP-3D set layout
__global__ void stream7(const float* __restrict__ P, const float* __restrict__ Q, const float* __restrict__ v,
                        float* __restrict__ Pn, int Z, size_t HW) {
    size_t n = (size_t)Z * HW;
    for (size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (size_t)gridDim.x * blockDim.x) {
        size_t z = o / HW, ij = o - z * HW;
        size_t b = ((z + 1) * 3) * HW + ij;
        float a0 = P[b], a1 = P[b + HW], a2 = P[b + 2 * HW];
        float q0 = Q[b], q1 = Q[b + HW], q2 = Q[b + 2 * HW];
        float vv = v[o];
        Pn[b] = a0 + q0 * vv; Pn[b + HW] = a1 + q1 * vv; Pn[b + 2 * HW] = a2 + q2 * vv;
    }
}
__global__ void stream7v4(const float4* __restrict__ P, const float4* __restrict__ Q, const float4* __restrict__ v,
                        float4* __restrict__ Pn, int Z, size_t HW4) {
    size_t n = (size_t)Z * HW4;
    for (size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (size_t)gridDim.x * blockDim.x) {
        size_t z = o / HW4, ij = o - z * HW4;
        size_t b = ((z + 1) * 3) * HW4 + ij;
        float4 a0 = P[b], a1 = P[b + HW4], a2 = P[b + 2 * HW4];
        float4 q0 = Q[b], q1 = Q[b + HW4], q2 = Q[b + 2 * HW4];
        float4 vv = v[o];
        a0.x += q0.x * vv.x; a0.y += q0.y * vv.y; a0.z += q0.z * vv.z; a0.w += q0.w * vv.w;
        a1.x += q1.x * vv.x; a1.y += q1.y; a1.z += q1.z; a1.w += q1.w;
        a2.x += q2.x; a2.y += q2.y; a2.z += q2.z; a2.w += q2.w;
        Pn[b] = a0; Pn[b + HW4] = a1; Pn[b + 2 * HW4] = a2;
    }
}
int main() {
    int Z = 256; size_t HW = 256 * 256;
    size_t set = (size_t)(Z + 2) * 3 * HW;
    float *work, *v;
    cudaMalloc(&work, 3 * set * 4); cudaMalloc(&v, Z * HW * 4);
    cudaMemset(work, 0, 3 * set * 4); cudaMemset(v, 0, Z * HW * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode)
    for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        for (int w = 0; w < 3; ++w) {
            if (mode == 0) stream7<<<blocks, 256>>>(work, work + set, v, work + 2 * set, Z, HW);
            else stream7v4<<<blocks, 256>>>((float4*)work, (float4*)(work + set), (float4*)v, (float4*)(work + 2 * set), Z, HW / 4);
        }
        cudaEventRecord(e0);
        for (int it = 0; it < 20; ++it) {
            const int k = it % 3;
            float* P = work + k * set; float* Q = work + ((k + 2) % 3) * set; float* Pn = work + ((k + 1) % 3) * set;
            if (mode == 0) stream7<<<blocks, 256>>>(P, Q, v, Pn, Z, HW);
            else stream7v4<<<blocks, 256>>>((float4*)P, (float4*)Q, (float4*)v, (float4*)Pn, Z, HW / 4);
        }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double us = ms * 1000 / 20;
        printf("mode %d blocks %d: %.1f us/iter, %.0f GB/s (40 B/voxel)\n", mode, blocks, us, 40.0 * Z * HW / us / 1e3);
    }
    return 0;
}
