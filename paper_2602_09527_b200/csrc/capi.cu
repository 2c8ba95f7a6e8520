// C ABI: plan / selection lifecycle, standalone operator entry points.
// See include/proxtomo_b200.h for the contract of every function.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <vector>

#include "pt_internal.cuh"

namespace pt {

static thread_local char g_err[1024] = "";
std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void workspace_sizes(const pt_plan* plan, size_t* partial_floats, size_t* red_doubles,
                     size_t* image_floats)
{
    *partial_floats =
        (size_t)plan->n_bands * plan->Z * plan->B * (size_t)plan->max_angles_per_launch;
    const size_t chunks = (plan->A + plan->max_angles_per_launch - 1) / plan->max_angles_per_launch;
    // block sums of the residual norm: one per 256 rows (band reduction) or
    // one per 32 rays (small-image forward)
    *red_doubles = ((size_t)plan->A * plan->Z * plan->B + 31) / 32 + chunks + 16;
    *image_floats = (size_t)plan->Z * plan->H * plan->W;
}

bool pdl_enabled()
{
    static const bool on = [] {
        const char* e = getenv("PT_PDL");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

typedef CUresult (*fn_encode_tiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static fn_encode_tiled encode_tiled()
{
    static fn_encode_tiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (fn_encode_tiled)p;
    }();
    return fn;
}

bool tma_available() { return encode_tiled() != nullptr; }

// float32 tensor of `rank` dims (innermost first, dense), box `box`; zero fill
// outside the tensor
int make_map(CUtensorMap* m, const float* base, int rank, const cuuint64_t* dims,
                    const cuuint32_t* box)
{
    fn_encode_tiled enc = encode_tiled();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return PT_ECUDA; }
    cuuint64_t strides[4];
    cuuint64_t acc = 4;
    for (int d = 0; d + 1 < rank; ++d) {
        acc *= dims[d];
        strides[d] = acc;
    }
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, (void*)base, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return PT_ECUDA; }
    return PT_OK;
}

int ensure_smem(const void* kernel, size_t bytes)
{
    if (bytes <= 48 * 1024) return PT_OK;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    PT_CHECK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = done[{kernel, dev}];
    if (have >= bytes) return PT_OK;
    PT_CHECK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)bytes));
    have = bytes;
    return PT_OK;
}

int workspace_alloc(const pt_plan* plan, Workspace* ws)
{
    workspace_sizes(plan, &ws->partial_floats, &ws->red_doubles, &ws->image_floats);
    PT_CHECK_CUDA(cudaMalloc(&ws->partial, ws->partial_floats * sizeof(float)));
    PT_CHECK_CUDA(cudaMalloc(&ws->red, ws->red_doubles * sizeof(double)));
    PT_CHECK_CUDA(cudaMalloc(&ws->image, ws->image_floats * sizeof(float)));
    return PT_OK;
}

void workspace_free(Workspace* ws)
{
    if (ws->partial) cudaFree(ws->partial);
    if (ws->red) cudaFree(ws->red);
    if (ws->image) cudaFree(ws->image);
    ws->partial = nullptr;
    ws->red = nullptr;
    ws->image = nullptr;
}

// Row slab: the grid is rows [row0, row0 + H) of an Hg-row image; positions
// are taken relative to the slab (row-stepping: step 0 is image row row0;
// column-stepping: lane 0 is image row row0).
static AngleTab make_tab(double theta, int Hg, int row0, int W, int B, double ds, double h)
{
    AngleTab t;
    const double c = cos(theta), s = sin(theta);
    const double cB = (B - 1) / 2.0, cH = (Hg - 1) / 2.0, cW = (W - 1) / 2.0;
    if (fabs(c) >= fabs(s)) {  // projector.py:32
        t.branch = 0;
        t.sigma = ds / (h * c);
        t.m = -(s / c);
        t.a0 = -cB * t.sigma + cH * (s / c) + cW;
        if (row0) t.a0 += t.m * row0;
        t.step_len = (float)(h / fabs(c));
    } else {
        t.branch = 1;
        t.sigma = ds / (h * s);
        t.m = -(c / s);
        t.a0 = -cB * t.sigma + cW * (c / s) + cH;
        if (row0) t.a0 -= row0;
        t.step_len = (float)(h / fabs(s));
    }
    t.isig = 1.0 / t.sigma;
    t.im = fabs(t.m) < 1e-300 ? 0.0 : 1.0 / t.m;
    // d(b, r, c) = sigma b + ar r + ac c + a0 (pos_b - lane); b_f solves d = 0
    const double ar = t.branch ? -1.0 : t.m, ac = t.branch ? t.m : -1.0;
    t.gbr = -ar / t.sigma;
    t.gbc = -ac / t.sigma;
    t.gg = -t.a0 / t.sigma;
    return t;
}

static int selection_build(pt_plan* plan, const int32_t* idx, int32_t n, pt_selection** out)
{
    pt_selection* sel = new pt_selection();
    sel->n = n;
    sel->h_angle.resize(n);
    std::vector<int32_t> br[2];
    for (int k = 0; k < n; ++k) {
        const int a = idx ? idx[k] : k;
        if (a < 0 || a >= plan->A) {
            delete sel;
            set_error("angle index out of range [0, %d)", plan->A);
            return PT_EINVAL;
        }
        sel->h_angle[k] = a;
        br[plan->h_tab[a].branch].push_back(k);
    }
    auto up = [&](int32_t** d, const std::vector<int32_t>& v) -> int {
        PT_CHECK_CUDA(cudaMalloc(d, std::max<size_t>(1, v.size()) * sizeof(int32_t)));
        if (!v.empty())
            PT_CHECK_CUDA(cudaMemcpy(*d, v.data(), v.size() * sizeof(int32_t),
                                     cudaMemcpyHostToDevice));
        return PT_OK;
    };
    int rc = up(&sel->d_angle, sel->h_angle);
    for (int b = 0; b < 2 && rc == PT_OK; ++b) {
        sel->n_branch[b] = (int32_t)br[b].size();
        rc = up(&sel->d_branch_pos[b], br[b]);
    }
    if (rc != PT_OK) {
        delete sel;
        return rc;
    }
    {
        std::lock_guard<std::mutex> g(plan->mu);
        plan->selections.push_back(sel);
    }
    *out = sel;
    return PT_OK;
}

}  // namespace pt

using namespace pt;

extern "C" {

const char* pt_last_error(void) { return g_err; }
const char* pt_version(void) { return "proxtomo_b200 0.1.0 sm_100a"; }
int64_t pt_launch_count(void) { return g_launches.load(); }
int64_t pt_geometry_desc_size(void) { return (int64_t)sizeof(pt_geometry_desc); }

int pt_plan_create(const pt_geometry_desc* d, pt_plan** out)
{
    if (!d || !out) { set_error("null argument"); return PT_EINVAL; }
    if (d->height < 1 || d->width < 1 || d->n_slices < 1) { set_error("grid must be positive"); return PT_EINVAL; }
    if (d->n_angles < 1) { set_error("geometry needs at least one projection angle"); return PT_EINVAL; }
    if (d->n_bins < 1) { set_error("n_bins must be >= 1"); return PT_EINVAL; }
    if (!(d->bin_spacing > 0.0) || !(d->pixel_size > 0.0)) {
        set_error("bin_spacing and pixel_size must be positive");
        return PT_EINVAL;
    }
    for (int a = 0; a < d->n_angles; ++a) {
        if (a && !(d->host_angles[a] > d->host_angles[a - 1])) { set_error("angles must be strictly increasing"); return PT_EINVAL; }
    }
    if (d->host_angles[0] < 0.0 || d->host_angles[d->n_angles - 1] >= M_PI) { set_error("angles must lie in [0, pi)"); return PT_EINVAL; }

    if (d->rows_total != 0 && (d->row_offset < 0 || d->rows_total < d->row_offset + d->height)) {
        set_error("row slab outside the image");
        return PT_EINVAL;
    }
    if (d->rows_total != 0 && d->n_slices != 1) { set_error("row slabs are 2D"); return PT_EINVAL; }

    pt_plan* p = new pt_plan();
    p->H = d->height; p->W = d->width; p->Z = d->n_slices;
    p->row0 = d->rows_total ? d->row_offset : 0;
    p->Hg = d->rows_total ? d->rows_total : d->height;
    p->A = d->n_angles; p->B = d->n_bins;
    p->ds = d->bin_spacing; p->h = d->pixel_size;
    p->angles.assign(d->host_angles, d->host_angles + d->n_angles);
    p->h_tab.resize(p->A);
    double max_br = 0, max_bc = 0, min_abs_sigma = 1e300;
    for (int a = 0; a < p->A; ++a) {
        const AngleTab t = make_tab(p->angles[a], p->Hg, p->row0, p->W, p->B, p->ds, p->h);
        p->h_tab[a] = t;
        const double ar = t.branch ? -1.0 : t.m, ac = t.branch ? t.m : -1.0;
        max_br = std::max(max_br, fabs(ar / t.sigma));
        max_bc = std::max(max_bc, fabs(ac / t.sigma));
        min_abs_sigma = std::min(min_abs_sigma, fabs(t.sigma));
    }
    p->cand_half = std::max(1, (int)ceil(1.0 / min_abs_sigma - 1e-12));
    const int mn = std::min(p->H, p->W);
    // forward tile configuration (band height TY x lane tile TX), see projector.cu
    static const int cfg_env = [] {
        const char* e = getenv("PT_FWD_CFG");
        return e ? atoi(e) : -1;
    }();
    // slice stacks (config 3: 256 slices of 256^2) have CTAs to spare: 64-step
    // bands on 128-lane tiles (c3 subset forward 122 -> 100 us against the
    // 32 x 128 tiles a single 256^2 image needs to fill the GPU)
    if (mn >= 512) p->fwd_cfg = 3;
    else if (mn >= 128) p->fwd_cfg = p->Z > 1 ? 1 : 100;
    else p->fwd_cfg = 101;
    if (cfg_env >= 0) p->fwd_cfg = cfg_env;  // PT_FWD_CFG overrides every size
    pt::forward_config(p->fwd_cfg, &p->fwd_ty, &p->fwd_tx);
    p->n_bands = (std::max(p->H, p->W) + p->fwd_ty - 1) / p->fwd_ty;
    const size_t per_angle = (size_t)p->n_bands * p->Z * p->B;
    const size_t cap_floats = (size_t)1 << 28;  // 1 GiB of band partials
    p->max_angles_per_launch = (int)std::max<size_t>(1, std::min<size_t>(p->A, cap_floats / per_angle));
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) { set_error("cudaGetDevice: %s", cudaGetErrorString(e)); delete p; return PT_ECUDA; }
    // gather tile: the largest whose CTA count still fills ~4 waves of SMs
    {
        static const int env = [] {
            const char* v = getenv("PT_GATHER_TILE");
            return v ? atoi(v) : -1;
        }();
        auto ctas = [&](int t) {
            return (long long)((p->W + kGatherTiles[t][1] - 1) / kGatherTiles[t][1]) *
                   ((p->H + kGatherTiles[t][0] - 1) / kGatherTiles[t][0]) * p->Z;
        };
        int pick = 2;
        for (int t = 0; t < 3; ++t) {
            if (ctas(t) >= 4LL * p->sm_count) { pick = t; break; }
        }
        // images too small to give every SM one 16 x 64 tile (config 0,
        // 128^2): 8 x 64 tiles (c0 4299 -> 4427 epochs/s; c1 keeps 16 x 64,
        // 1598 vs 1545)
        if (pick == 2 && ctas(2) < p->sm_count) pick = 3;
        p->gather_tile = (env >= 0 && env < 4) ? env : pick;
        const int tr = kGatherTiles[p->gather_tile][0], tc = kGatherTiles[p->gather_tile][1];
        p->gather_slot = (int)ceil((tr - 1) * max_br + (tc - 1) * max_bc) + 2 * p->cand_half + 8;
    }
    if (cudaMalloc(&p->d_tab, sizeof(AngleTab) * p->A) != cudaSuccess ||
        cudaMemcpy(p->d_tab, p->h_tab.data(), sizeof(AngleTab) * p->A, cudaMemcpyHostToDevice) != cudaSuccess) {
        set_error("angle table upload failed");
        delete p;
        return PT_ECUDA;
    }
    int rc = workspace_alloc(p, &p->ws);
    if (rc == PT_OK) rc = selection_build(p, nullptr, p->A, &p->all);
    if (rc != PT_OK) { pt_plan_destroy(p); return rc; }
    *out = p;
    return PT_OK;
}

int pt_plan_destroy(pt_plan* p)
{
    if (!p) return PT_OK;
    for (pt_selection* s : p->selections) {
        cudaFree(s->d_angle);
        cudaFree(s->d_branch_pos[0]);
        cudaFree(s->d_branch_pos[1]);
        delete s;
    }
    workspace_free(&p->ws);
    if (p->d_tab) cudaFree(p->d_tab);
    delete p;
    return PT_OK;
}

int pt_selection_create(pt_plan* plan, const int32_t* host_idx, int32_t n, pt_selection** out)
{
    if (!plan || !out) { set_error("null argument"); return PT_EINVAL; }
    if (!host_idx && n == -1) { *out = plan->all; return PT_OK; }
    if (n < 0 || (!host_idx && n > 0)) { set_error("bad selection"); return PT_EINVAL; }
    return selection_build(plan, host_idx, n, out);
}

int32_t pt_selection_size(const pt_selection* sel) { return sel ? sel->n : -1; }

int64_t pt_selection_nnz(pt_plan* plan, const pt_selection* sel)
{
    if (!plan || !sel) return -1;
    if (sel->nnz >= 0) return sel->nnz;
    // exact count of kept COO entries (projector.py:55-60), float64 as the reference
    int64_t total = 0;
    // image rows [r_lo, r_hi) are this plan's (a row slab counts its own taps)
    const int H = plan->Hg, W = plan->W, B = plan->B;
    const int r_lo = plan->row0, r_hi = plan->row0 + plan->H;
    for (int k = 0; k < sel->n; ++k) {
        const double th = plan->angles[sel->h_angle[k]];
        const double c = cos(th), s = sin(th), h = plan->h;
        const bool rows = fabs(c) >= fabs(s);
        const int st_lo = rows ? r_lo : 0, st_hi = rows ? r_hi : W;
        const int n_lanes = rows ? W : H;
        const int ln_lo = rows ? 0 : r_lo, ln_hi = rows ? W : r_hi;
        const double step_len = rows ? h / fabs(c) : h / fabs(s);
        int64_t cnt = 0;
#pragma omp parallel for reduction(+ : cnt)
        for (int b = 0; b < B; ++b) {
            const double sb = ((double)b - (B - 1) / 2.0) * plan->ds;
            for (int st = st_lo; st < st_hi; ++st) {
                double cross;
                if (rows) cross = (sb - (((double)st - (H - 1) / 2.0) * h) * s) / c;
                else cross = (sb - (((double)st - (W - 1) / 2.0) * h) * c) / s;
                const double pos = cross / h + (n_lanes - 1) / 2.0;
                const double fl = floor(pos);
                const double fr = pos - fl;
                const long long l0 = (long long)fl;
                if (l0 >= ln_lo && l0 < ln_hi && (1.0 - fr) * step_len > 0.0) ++cnt;
                if (l0 + 1 >= ln_lo && l0 + 1 < ln_hi && fr * step_len > 0.0) ++cnt;
            }
        }
        total += cnt;
    }
    const_cast<pt_selection*>(sel)->nnz = total * plan->Z;
    return sel->nnz;
}

int pt_forward(pt_plan* plan, const pt_selection* sel, const float* x, const float* x2,
               const float* data, float* y, double* sumsq, void* stream)
{
    if (!plan || !sel || !x || !y) { set_error("null argument"); return PT_EINVAL; }
    return launch_forward(plan, &plan->ws, sel, x, x2, data, y, sumsq, (cudaStream_t)stream);
}

int pt_adjoint(pt_plan* plan, const pt_selection* sel, const float* y, float* x_out, float alpha,
               int32_t accumulate, void* stream)
{
    if (!plan || !sel || !y || !x_out) { set_error("null argument"); return PT_EINVAL; }
    if (sel->n == 0) {
        if (!accumulate)
            PT_CHECK_CUDA(cudaMemsetAsync(x_out, 0, sizeof(float) * (size_t)plan->Z * plan->H * plan->W,
                                          (cudaStream_t)stream));
        return PT_OK;
    }
    return launch_adjoint(plan, sel, y, x_out, alpha, accumulate, nullptr, (cudaStream_t)stream);
}

static int check_ep(const pt_step_epilogue* ep)
{
    if (!ep || !ep->x || !ep->h) { set_error("epilogue needs x and h"); return PT_EINVAL; }
    if (ep->estimator < PT_EST_FULL || ep->estimator > PT_EST_LSVRG) { set_error("unknown estimator"); return PT_EINVAL; }
    if (ep->estimator == PT_EST_SAGA && (!ep->aux0 || !ep->aux1)) { set_error("saga needs table and sum"); return PT_EINVAL; }
    if ((ep->estimator == PT_EST_SVRG || ep->estimator == PT_EST_LSVRG) && !ep->aux0) { set_error("svrg needs full_grad"); return PT_EINVAL; }
    if (ep->theta ? (!ep->v_out || !ep->xhat_out) : !ep->x_out) { set_error("missing epilogue output"); return PT_EINVAL; }
    return PT_OK;
}

int pt_adjoint_step(pt_plan* plan, const pt_selection* sel, const float* r,
                    const pt_step_epilogue* ep, void* stream)
{
    if (!plan || !sel || !r) { set_error("null argument"); return PT_EINVAL; }
    int rc = check_ep(ep);
    if (rc) return rc;
    return launch_adjoint(plan, sel, r, nullptr, 1.f, 0, ep, (cudaStream_t)stream);
}

int pt_step_epilogue_apply(pt_plan* plan, const float* g, const pt_step_epilogue* ep, void* stream)
{
    if (!plan || !g) { set_error("null argument"); return PT_EINVAL; }
    int rc = check_ep(ep);
    if (rc) return rc;
    return launch_epilogue(plan, g, ep, (cudaStream_t)stream);
}

int64_t pt_fgp_workspace_floats(pt_plan* plan) { return plan ? fgp_workspace_floats(plan) : -1; }

int pt_tv_prox(pt_plan* plan, const float* v, double lam, int32_t inner_iterations, int32_t nonneg,
               float* p, float* q, float* w, float* x_out, const float* xhat, float* h,
               float p_over_gamma, int64_t iteration, int64_t* bad_iter, float* work, void* stream)
{
    if (!plan || !v || !p || !q || !x_out || !work) { set_error("null argument"); return PT_EINVAL; }
    if (plan->Z > 1 && !w) { set_error("3D prox needs the third dual"); return PT_EINVAL; }
    if (!(lam > 0.0)) { set_error("tau must be positive"); return PT_EINVAL; }
    if (h && !xhat) { set_error("h update needs x_hat"); return PT_EINVAL; }
    return launch_tv_prox(plan, v, lam, inner_iterations, nonneg, p, q, w, x_out, xhat, h,
                          p_over_gamma, iteration, bad_iter, work, (cudaStream_t)stream);
}

int pt_tv_prox_emulate_rows(pt_plan* plan, int32_t slabs, const float* v, double lam,
                            int32_t inner_iterations, int32_t nonneg, float* p, float* q,
                            float* x_out, void* stream)
{
    if (!plan || !v || !p || !q || !x_out) { set_error("null argument"); return PT_EINVAL; }
    if (plan->Z != 1) { set_error("row slabs are a 2D decomposition"); return PT_EINVAL; }
    if (!(lam > 0.0)) { set_error("tau must be positive"); return PT_EINVAL; }
    if (slabs < 1 || slabs > plan->H) { set_error("bad slab count"); return PT_EINVAL; }
    cudaStream_t st = (cudaStream_t)stream;
    const int H = plan->H, W = plan->W;
    std::vector<Fgp2Slab> sl(slabs);
    size_t total = 0;
    for (int g = 0; g < slabs; ++g) {
        sl[g].r0 = (int)((long long)H * g / slabs);
        sl[g].Hl = (int)((long long)H * (g + 1) / slabs) - sl[g].r0;
        total += (size_t)fgp2d_slab_floats(sl[g].Hl, W);
    }
    float* work = nullptr;
    PT_CHECK_CUDA(cudaMallocAsync(&work, total * 4, st));
    float* w = work;
    for (int g = 0; g < slabs; ++g) {
        const size_t off = (size_t)sl[g].r0 * W;
        sl[g].v = v + off; sl[g].p = p + off; sl[g].q = q + off; sl[g].x_out = x_out + off;
        sl[g].work = w;
        w += fgp2d_slab_floats(sl[g].Hl, W);
    }
    const int rc = fgp2d_rows_run(sl.data(), slabs, H, W, lam, inner_iterations, nonneg, 0.f, 0,
                                  nullptr, nullptr, st);
    cudaFreeAsync(work, st);
    return rc;
}

int pt_dot(const float* a, const float* b, int64_t n, double* out, void* stream)
{
    if (!a || !b || !out || n < 0) { set_error("bad argument"); return PT_EINVAL; }
    return launch_dot(a, b, n, out, (cudaStream_t)stream);
}

int pt_tv_value(pt_plan* plan, const float* x, double* out, void* stream)
{
    if (!plan || !x || !out) { set_error("null argument"); return PT_EINVAL; }
    return launch_tv_value(plan, x, out, (cudaStream_t)stream);
}

int pt_diff_norms(const float* x, const float* ref, int64_t n, double* out, void* stream)
{
    if (!x || !ref || !out || n < 0) { set_error("bad argument"); return PT_EINVAL; }
    return launch_diff_norms(x, ref, n, out, (cudaStream_t)stream);
}

int pt_operator_norm_sq(pt_plan* plan, float* v0, int32_t iterations, double* host_out, void* stream)
{
    if (!plan || !v0 || !host_out) { set_error("null argument"); return PT_EINVAL; }
    if (iterations < 1) { set_error("iterations must be >= 1"); return PT_EINVAL; }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)plan->Z * plan->H * plan->W;
    const size_t m = (size_t)plan->A * plan->Z * plan->B;
    float *y = nullptr, *u = nullptr;
    double* red = nullptr;
    double* hist = nullptr;
    int rc = PT_OK;
    std::vector<double> h(3 * (size_t)iterations);
    if (cudaMalloc(&y, m * 4) != cudaSuccess || cudaMalloc(&u, n * 4) != cudaSuccess ||
        cudaMalloc(&red, 3 * PT_RED_DOUBLES * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&hist, 3 * (size_t)iterations * sizeof(double)) != cudaSuccess) {
        set_error("operator_norm_sq: allocation failed");
        rc = PT_ECUDA;
    }
    for (int it = 0; it < iterations && rc == PT_OK; ++it) {
        rc = launch_forward(plan, &plan->ws, plan->all, v0, nullptr, nullptr, y, nullptr, st);
        if (!rc) rc = launch_adjoint(plan, plan->all, y, u, 1.f, 0, nullptr, st);
        if (!rc) rc = launch_dot(v0, u, n, red, st);
        if (!rc) rc = launch_dot(v0, v0, n, red + PT_RED_DOUBLES, st);
        if (!rc) rc = launch_dot(u, u, n, red + 2 * PT_RED_DOUBLES, st);
        if (!rc) {
            for (int j = 0; j < 3; ++j)
                if (cudaMemcpyAsync(hist + 3 * it + j, red + j * PT_RED_DOUBLES, 8,
                                    cudaMemcpyDeviceToDevice, st) != cudaSuccess) rc = PT_ECUDA;
        }
        if (!rc) rc = launch_scale_by_rsqrt(v0, u, red + 2 * PT_RED_DOUBLES, n, st);
    }
    if (rc == PT_OK) {
        if (cudaMemcpyAsync(h.data(), hist, h.size() * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            set_error("operator_norm_sq: %s", cudaGetErrorString(cudaGetLastError()));
            rc = PT_ECUDA;
        }
    }
    if (rc == PT_OK) {
        // projector.py:170-180, replayed on the recorded scalars
        double est = 0.0;
        for (int it = 0; it < iterations; ++it) {
            est = h[3 * it] / h[3 * it + 1];
            if (sqrt(h[3 * it + 2]) == 0.0) { est = 0.0; break; }
        }
        *host_out = est;
    }
    cudaStreamSynchronize(st);
    if (y) cudaFree(y);
    if (u) cudaFree(u);
    if (red) cudaFree(red);
    if (hist) cudaFree(hist);
    return rc;
}

}  // extern "C"
