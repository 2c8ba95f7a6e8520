// Deterministic reductions (fixed grid, fixed combine order, float64
// accumulation) and small elementwise helpers.
//  - dot / sum of squares: power method (projector.py:170-180), objective
//    (solvers.py:271-277), relative error (metrics.py relative_error_sq)
//  - tv_value: regularizers.py:79-82 (isotropic, forward differences)
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "pt_internal.cuh"

namespace pt {

static constexpr int kRedBlocks = PT_RED_DOUBLES - 1;  // partials in out[1..]

__device__ __forceinline__ double block_sum(double v, double* sh)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
    return t;
}

__global__ void sum_doubles_kernel(const double* in, int64_t n, double* out, int accumulate)
{
    __shared__ double sh[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += in[i];
    double t = block_sum(s, sh);
    if (threadIdx.x == 0) {
        if (accumulate) *out += t; else *out = t;
    }
}

int launch_sum_doubles(const double* in, int64_t n, double* out, int accumulate, cudaStream_t st)
{
    sum_doubles_kernel<<<1, 1024, 0, st>>>(in, n, out, accumulate);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

__global__ void dot_kernel(const float* a, const float* b, int64_t n, double* part)
{
    __shared__ double sh[32];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        s += (double)a[i] * (double)b[i];
    double t = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

static int grid_for(int64_t n)
{
    return (int)std::max<int64_t>(1, std::min<int64_t>(kRedBlocks, (n + 255) / 256));
}

int launch_dot(const float* a, const float* b, int64_t n, double* out, cudaStream_t st)
{
    const int g = grid_for(n);
    dot_kernel<<<g, 256, 0, st>>>(a, b, n, out + 1);
    PT_CHECK_LAUNCH();
    return launch_sum_doubles(out + 1, g, out, 0, st);
}

__global__ void diff_norms_kernel(const float* x, const float* ref, int64_t n, double* part)
{
    __shared__ double sh[32];
    double d = 0.0, r = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double xr = ref[i];
        const double df = (double)x[i] - xr;
        d += df * df;
        r += xr * xr;
    }
    double t = block_sum(d, sh);
    __syncthreads();
    double u = block_sum(r, sh);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = t;
        part[gridDim.x + blockIdx.x] = u;
    }
}

int launch_diff_norms(const float* x, const float* ref, int64_t n, double* out, cudaStream_t st)
{
    // out[0], out[1] results; partials in out[2 ..]
    const int g = std::min(grid_for(n), (kRedBlocks - 1) / 2);
    diff_norms_kernel<<<g, 256, 0, st>>>(x, ref, n, out + 2);
    PT_CHECK_LAUNCH();
    int rc = launch_sum_doubles(out + 2, g, out, 0, st);
    if (rc) return rc;
    return launch_sum_doubles(out + 2 + g, g, out + 1, 0, st);
}

__global__ void tv_kernel(const float* x, int Z, int H, int W, double* part)
{
    __shared__ double sh[32];
    const int64_t plane = (int64_t)H * W;
    const int64_t n = plane * Z;
    double s = 0.0;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(o % W);
        const int64_t t1 = o / W;
        const int i = (int)(t1 % H);
        const int k = (int)(t1 / H);
        const double xo = x[o];
        const double gv = (i < H - 1) ? (double)x[o + W] - xo : 0.0;
        const double gh = (j < W - 1) ? (double)x[o + 1] - xo : 0.0;
        const double gz = (Z > 1 && k < Z - 1) ? (double)x[o + plane] - xo : 0.0;
        s += sqrt(gv * gv + gh * gh + gz * gz);
    }
    double t = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

int launch_tv_value(const pt_plan* plan, const float* x, double* out, cudaStream_t st)
{
    const int64_t n = (int64_t)plan->Z * plan->H * plan->W;
    const int g = grid_for(n);
    tv_kernel<<<g, 256, 0, st>>>(x, plan->Z, plan->H, plan->W, out + 1);
    PT_CHECK_LAUNCH();
    return launch_sum_doubles(out + 1, g, out, 0, st);
}

// Identity prox (problem without a regulariser, solvers.py:227) fused with the
// control-variate update h += (p/gamma)(x+ - x_hat) (solvers.py:249-250).
__global__ void identity_prox_kernel(const float* v, const float* xhat, float* x_out, float* h,
                                     float pog, int64_t n, long long iteration,
                                     long long* bad_iter)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float x = v[i];
        x_out[i] = x;
        if (h) h[i] = h[i] + pog * (x - xhat[i]);
        if (!isfinite(x) && bad_iter) atomicMin(bad_iter, iteration);
    }
}

int launch_identity_prox(const float* v, const float* xhat, float* x_out, float* h,
                         float p_over_gamma, int64_t n, int64_t iteration, int64_t* bad_iter,
                         cudaStream_t st)
{
    const int g = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    identity_prox_kernel<<<g, 256, 0, st>>>(v, xhat, x_out, h, p_over_gamma, n,
                                            (long long)iteration, (long long*)bad_iter);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

// v = u / sqrt(sumsq[0])   (projector.py:180, v = u / norm)
__global__ void scale_rsqrt_kernel(float* v, const float* u, const double* sumsq, int64_t n)
{
    const double nrm = sqrt(*sumsq);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (float)((double)u[i] * inv);
}

int launch_scale_by_rsqrt(float* v, const float* u, const double* sumsq, int64_t n,
                          cudaStream_t st)
{
    const int g = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    scale_rsqrt_kernel<<<g, 256, 0, st>>>(v, u, sumsq, n);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

// FISTA momentum (solvers.py:384-386): x+ = src (the prox output, or the
// prox input when there is no regulariser), y = x+ + beta (x+ - x); a
// non-finite x+ lowers *bad_iter (solvers.py:380-381).
__global__ void fista_momentum_kernel(const float* src, const float* x_prev, float* x_out,
                                      float* y, float beta, int64_t n, long long iteration,
                                      long long* bad_iter)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float xn = src[i];
        if (x_out != src) x_out[i] = xn;
        y[i] = xn + beta * (xn - x_prev[i]);
        if (!isfinite(xn)) atomicMin(bad_iter, iteration);
    }
}

int launch_fista_momentum(const float* src, const float* x_prev, float* x_out, float* y,
                          float beta, int64_t n, int64_t iteration, int64_t* bad_iter,
                          cudaStream_t st)
{
    const int g = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    fista_momentum_kernel<<<g, 256, 0, st>>>(src, x_prev, x_out, y, beta, n,
                                             (long long)iteration, (long long*)bad_iter);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

__global__ void fill_i64_kernel(int64_t* p, int64_t value) { *p = value; }

int launch_fill_i64(int64_t* p, int64_t value, cudaStream_t st)
{
    fill_i64_kernel<<<1, 1, 0, st>>>(p, value);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

}  // namespace pt
