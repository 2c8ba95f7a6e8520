// Diagonally preconditioned primal-dual (PDHG) reference solver, device side
// (solvers.py:395-455).  The projector calls come from the existing forward
// (with the data subtraction fused) and gather adjoint; these are the three
// elementwise steps of one iteration, each one pass over its arrays:
//   dual_sino : y  = (y + sigma_a (A xbar - b)) / (1 + sigma_a)        (:434)
//   dual_tv   : z  = clip_alpha(z + sigma_d D xbar)                    (:436-442)
//   primal    : x' = max(x - tau (A^T y + D^T z), 0); xbar = 2 x' - x  (:443-451)
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "pt_internal.cuh"

namespace pt {

static int grid1d(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

__global__ void pdhg_dual_sino_kernel(float* y, const float* resid, const float* sigma_a, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float s = sigma_a[i];
        y[i] = (y[i] + s * resid[i]) / (1.f + s);
    }
}

// one (H, W) plane per blockIdx.y; forward differences, zero on the last row / column
__global__ void pdhg_dual_tv_kernel(const float* xbar, float* zv, float* zh, int H, int W,
                                    float sigma_d, float inv_alpha)
{
    const int64_t plane = (int64_t)H * W;
    const int64_t base = (int64_t)blockIdx.y * plane;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < plane;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(o / W), j = (int)(o - (int64_t)i * W);
        const int64_t g = base + o;
        const float xo = xbar[g];
        const float gv = (i < H - 1) ? xbar[g + W] - xo : 0.f;
        const float gh = (j < W - 1) ? xbar[g + 1] - xo : 0.f;
        const float a = zv[g] + sigma_d * gv;
        const float b = zh[g] + sigma_d * gh;
        const float scale = fmaxf(1.f, sqrtf(a * a + b * b) * inv_alpha);
        zv[g] = a / scale;
        zh[g] = b / scale;
    }
}

__global__ void pdhg_primal_kernel(float* x, float* xbar, const float* ascent, const float* zv,
                                   const float* zh, const float* tau, int H, int W, int use_tv,
                                   int nonneg, long long iteration, long long* bad_iter)
{
    const int64_t plane = (int64_t)H * W;
    const int64_t base = (int64_t)blockIdx.y * plane;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < plane;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(o / W), j = (int)(o - (int64_t)i * W);
        const int64_t g = base + o;
        float asc = ascent[g];
        if (use_tv) {
            // D^T(a, b) = -a[i]·[i<H-1] + a[i-1]·[i>0] - b[j]·[j<W-1] + b[j-1]·[j>0]
            float d = (i < H - 1) ? -zv[g] : 0.f;
            if (i > 0) d += zv[g - W];
            if (j < W - 1) d -= zh[g];
            if (j > 0) d += zh[g - 1];
            asc += d;
        }
        const float xo = x[g];
        float xn = xo - tau[g] * asc;
        if (nonneg) xn = fmaxf(xn, 0.f);
        x[g] = xn;
        xbar[g] = 2.f * xn - xo;
        if (!isfinite(xn) && bad_iter) atomicMin(bad_iter, iteration);
    }
}

}  // namespace pt

using namespace pt;

extern "C" {

int pt_pdhg_dual_sino(float* y, const float* resid, const float* sigma_a, int64_t n, void* stream)
{
    if (!y || !resid || !sigma_a || n < 0) { set_error("bad argument"); return PT_EINVAL; }
    if (n == 0) return PT_OK;
    pdhg_dual_sino_kernel<<<grid1d(n), 256, 0, (cudaStream_t)stream>>>(y, resid, sigma_a, n);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

int pt_pdhg_dual_tv(const float* xbar, float* zv, float* zh, int32_t n_slices, int32_t height,
                    int32_t width, double sigma_d, double alpha, void* stream)
{
    if (!xbar || !zv || !zh || n_slices < 1 || height < 1 || width < 1 || !(alpha > 0.0)) {
        set_error("bad argument");
        return PT_EINVAL;
    }
    const int64_t plane = (int64_t)height * width;
    dim3 grid(grid1d(plane), n_slices);
    pdhg_dual_tv_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        xbar, zv, zh, height, width, (float)sigma_d, (float)(1.0 / alpha));
    PT_CHECK_LAUNCH();
    return PT_OK;
}

int pt_pdhg_primal(float* x, float* xbar, const float* ascent, const float* zv, const float* zh,
                   const float* tau, int32_t n_slices, int32_t height, int32_t width,
                   int32_t nonneg, int64_t iteration, int64_t* bad_iter, void* stream)
{
    const int use_tv = zv != nullptr;
    if (!x || !xbar || !ascent || !tau || (use_tv && !zh) || n_slices < 1 || height < 1 ||
        width < 1) {
        set_error("bad argument");
        return PT_EINVAL;
    }
    const int64_t plane = (int64_t)height * width;
    dim3 grid(grid1d(plane), n_slices);
    pdhg_primal_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        x, xbar, ascent, zv, zh, tau, height, width, use_tv, nonneg, (long long)iteration,
        (long long*)bad_iter);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

}  // extern "C"
