// Matrix-free Joseph projector for sm_100a: forward (band-tiled, smem-staged)
// and adjoint (pixel-driven gather with the estimator/ProxSkip epilogue fused).
//
// Reference semantics: pkg/src/proxtomo/projector.py:26-61 (weights),
// :114-126 (forward, subset rows in subset order), :129-140 (adjoint).
// See DESIGN.md for the tiling, the precision argument and the roofline.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "pt_internal.cuh"

namespace pt {

// floor() on the fma pipe: x + 1.5*2^23 rounded toward -inf leaves floor(x)
// in the low mantissa bits (valid for |x| < 2^22).
static constexpr float kMagic = 12582912.0f;
static constexpr int kMagicBits = 0x4B400000;

// ---------------------------------------------------------------------------
// Forward: one CTA = one band of TY consecutive steps (image rows for
// row-stepping angles, image columns for column-stepping ones) x one tile of
// TX lanes, staged once in shared memory (transposed for the column branch so
// both branches read lanes contiguously).  The CTA then walks every selected
// angle of its branch and, for each ray it owns (ray position at the band's
// middle step inside [l0, l0+TX); the edge tiles also own the rays beyond),
// sums the <= TY Joseph samples of that ray inside the band.  Each
// (band, ray) partial is written exactly once, so the band reduction that
// follows is deterministic and needs no atomics.  Partial sums of <= 64
// samples are combined in float64 (blocked fp32 sums).
// ---------------------------------------------------------------------------
struct FwdArgs {
    const float* x;
    const float* x2;
    float* partial;
    const AngleTab* tab;
    const int32_t* sel_angle;
    const int32_t* bpos0;
    const int32_t* bpos1;
    int32_t bbeg[2], bend[2];
    int32_t k_begin, n_k;
    int32_t H, W, Z, B;
    int32_t n_groups;
    int32_t n_bands;  // bands per slice in grid.y (max over branches)
};

template <int TY, int TX>
struct FwdTile {
    static constexpr int HL = TY / 2 + 3;
    static constexpr int PITCH = ((TX + 2 * HL) | 1);
    static constexpr int SMEM = TY * PITCH * 4;
};

template <int TY, int TX, int NT>
__global__ void __launch_bounds__(NT) fwd_band_kernel(FwdArgs P)
{
    using T = FwdTile<TY, TX>;
    extern __shared__ float sm[];
    constexpr int CH = 32;
    __shared__ int s_pref[CH + 1];
    __shared__ int s_blo[CH];
    __shared__ int s_k[CH];
    __shared__ double s_a0[CH], s_sig[CH], s_m[CH];

    const int branch = blockIdx.z & 1;
    const int group = blockIdx.z >> 1;
    const int band = blockIdx.y % P.n_bands;
    const int z = blockIdx.y / P.n_bands;
    const int n_steps = branch ? P.W : P.H;
    const int n_lanes = branch ? P.H : P.W;
    const int s0 = band * TY;
    const int l0 = blockIdx.x * TX;
    if (s0 >= n_steps || l0 >= n_lanes) return;
    const int bb = branch ? P.bbeg[1] : P.bbeg[0];
    const int nb = (branch ? P.bend[1] : P.bend[0]) - bb;
    const int a_begin = bb + (int)(((long long)nb * group) / P.n_groups);
    const int a_end = bb + (int)(((long long)nb * (group + 1)) / P.n_groups);
    if (a_begin >= a_end) return;
    const int32_t* bpos = branch ? P.bpos1 : P.bpos0;

    const int tid = threadIdx.x;
    const int lane_org = l0 - T::HL;
    const int ty_valid = min(TY, n_steps - s0);
    const size_t plane = (size_t)P.H * P.W;
    const float* img = P.x + (size_t)z * plane;
    const float* img2 = P.x2 ? P.x2 + (size_t)z * plane : nullptr;

    // ---- stage the tile (zero outside the image) ----
    if (branch == 0) {
        for (int idx = tid; idx < TY * T::PITCH; idx += NT) {
            int st = idx / T::PITCH, ll = idx - st * T::PITCH;
            int r = s0 + st, c = lane_org + ll;
            float v = 0.f;
            if (r < P.H && c >= 0 && c < P.W) {
                size_t o = (size_t)r * P.W + c;
                v = __ldg(img + o);
                if (img2) v -= __ldg(img2 + o);
            }
            sm[idx] = v;
        }
    } else {
        for (int idx = tid; idx < TY * T::PITCH; idx += NT) {
            int ll = idx / TY, st = idx - ll * TY;
            int r = lane_org + ll, c = s0 + st;
            float v = 0.f;
            if (c < P.W && r >= 0 && r < P.H) {
                size_t o = (size_t)r * P.W + c;
                v = __ldg(img + o);
                if (img2) v -= __ldg(img2 + o);
            }
            sm[st * T::PITCH + ll] = v;
        }
    }
    __syncthreads();

    const bool first_tile = (l0 == 0);
    const bool last_tile = (l0 + TX >= n_lanes);
    const double smid = s0 + 0.5 * (ty_valid - 1);

    for (int cbeg = a_begin; cbeg < a_end; cbeg += CH) {
        const int nc = min(CH, a_end - cbeg);
        if (tid < CH) {
            int cnt = 0;
            if (tid < nc) {
                const int k = bpos[cbeg + tid];
                const AngleTab t = P.tab[P.sel_angle[k]];
                // rays owned by this tile: pos at the middle step in [lo, hi)
                const double base = t.a0 + smid * t.m;
                long long blo, bhi;
                if (t.sigma > 0) {
                    blo = first_tile ? 0 : (long long)ceil(((double)l0 - base) / t.sigma);
                    bhi = last_tile ? P.B : (long long)ceil(((double)(l0 + TX) - base) / t.sigma);
                } else {
                    blo = last_tile ? 0 : (long long)floor(((double)(l0 + TX) - base) / t.sigma) + 1;
                    bhi = first_tile ? P.B : (long long)floor(((double)l0 - base) / t.sigma) + 1;
                }
                blo = max(blo, 0LL);
                bhi = min(bhi, (long long)P.B);
                cnt = (int)max(0LL, bhi - blo);
                s_blo[tid] = (int)blo;
                s_k[tid] = k;
                s_a0[tid] = t.a0;
                s_sig[tid] = t.sigma;
                s_m[tid] = t.m;
            }
            // inclusive warp scan of counts
            int v = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int n = __shfl_up_sync(0xffffffffu, v, o);
                if (tid >= o) v += n;
            }
            s_pref[tid + 1] = v;
            if (tid == 0) s_pref[0] = 0;
        }
        __syncthreads();
        const int total = s_pref[nc];
        int j = 0;
        for (int w = tid; w < total; w += NT) {
            while (w >= s_pref[j + 1]) ++j;
            const int b = s_blo[j] + (w - s_pref[j]);
            const double m = s_m[j];
            // global lane position at st = 0, then local (tile) coordinate
            const double P0 = s_a0[j] + (double)b * s_sig[j] + (double)s0 * m;
            // steps where pos in [-1.5, n_lanes + 0.5]: outside, both taps are zero
            int st_a = 0, st_b = ty_valid;
            if (fabs(m) < 1e-300) {
                if (P0 < -1.5 || P0 > n_lanes + 0.5) st_b = 0;
            } else {
                double e1 = (-1.5 - P0) / m, e2 = ((double)n_lanes + 0.5 - P0) / m;
                double lo = fmin(e1, e2), hi = fmax(e1, e2);
                st_a = max(st_a, (int)ceil(fmin(fmax(lo, -1.0), (double)TY + 1.0)));
                st_b = min(st_b, (int)floor(fmin(fmax(hi, -2.0), (double)TY + 1.0)) + 1);
            }
            const float pl = (float)(P0 - (double)lane_org);
            const float mf = (float)m;
            float acc = 0.f;
            for (int st = st_a; st < st_b; ++st) {
                const float pos = fmaf((float)st, mf, pl);
                const float tt = __fadd_rd(pos, kMagic);
                const int l = __float_as_int(tt) - kMagicBits;
                const float fr = pos - (tt - kMagic);
                const float* row = sm + st * T::PITCH + l;
                const float x0 = row[0], x1 = row[1];
                acc += fmaf(fr, x1 - x0, x0);
            }
            const size_t kk = (size_t)(s_k[j] - P.k_begin);
            P.partial[(((size_t)band * P.n_k + kk) * P.Z + z) * P.B + b] = acc;
        }
        __syncthreads();
    }
}

struct RedArgs {
    const float* partial;
    const AngleTab* tab;
    const int32_t* sel_angle;
    int32_t k_begin, n_k, Z, B;
    int32_t nb_row, nb_col;
    const float* data;
    float* y;
    double* block_sums;
};

__global__ void __launch_bounds__(256) fwd_reduce_kernel(RedArgs P)
{
    const size_t total = (size_t)P.n_k * P.Z * P.B;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (idx < total) {
        const int b = (int)(idx % P.B);
        const size_t t = idx / P.B;
        const int z = (int)(t % P.Z);
        const int kk = (int)(t / P.Z);
        const int k = kk + P.k_begin;
        const int ang = P.sel_angle[k];
        const AngleTab at = P.tab[ang];
        const int nb = at.branch ? P.nb_col : P.nb_row;
        const size_t stride = (size_t)P.n_k * P.Z * P.B;
        double s = 0.0;
        for (int band = 0; band < nb; ++band) s += (double)P.partial[band * stride + idx];
        float yv = (float)(s * (double)at.step_len);
        if (P.data) yv -= P.data[((size_t)ang * P.Z + z) * P.B + b];
        P.y[((size_t)k * P.Z + z) * P.B + b] = yv;
        sq = (double)yv * (double)yv;
    }
    if (P.block_sums) {
        __shared__ double red[8];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int i = 0; i < 8; ++i) s += red[i];
            P.block_sums[blockIdx.x] = s;
        }
    }
}

template <int TY, int TX, int NT>
static int run_forward_cfg(pt_plan* plan, Workspace* ws, const pt_selection* sel,
                           const float* x, const float* x2, const float* data, float* y,
                           double* sumsq, cudaStream_t st)
{
    using T = FwdTile<TY, TX>;
    static bool attr_set = false;
    if (!attr_set) {
        PT_CHECK_CUDA(cudaFuncSetAttribute(fwd_band_kernel<TY, TX, NT>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM));
        attr_set = true;
    }
    const int nb_row = (plan->H + TY - 1) / TY;
    const int nb_col = (plan->W + TY - 1) / TY;
    const int n_bands = plan->n_bands;
    const int n_tiles = (std::max(plan->H, plan->W) + TX - 1) / TX;
    const int n_chunk = std::max(1, plan->max_angles_per_launch);
    const size_t per_angle = (size_t)n_bands * plan->Z * plan->B;
    const int n_sel = sel->n;
    // prefix counts of branch members per selection slot, to slice the lists
    int n_blocks_red_total = 0;
    for (int kb = 0; kb < n_sel; kb += n_chunk) {
        int ke = std::min(n_sel, kb + n_chunk);
        n_blocks_red_total += (int)(((size_t)(ke - kb) * plan->Z * plan->B + 255) / 256);
    }
    if (sumsq && (size_t)n_blocks_red_total > ws->red_doubles) {
        set_error("reduction scratch too small");
        return PT_EINVAL;
    }
    int red_off = 0;
    int bi0 = 0, bi1 = 0;  // running positions in the branch lists
    for (int kb = 0; kb < n_sel; kb += n_chunk) {
        const int ke = std::min(n_sel, kb + n_chunk);
        if ((size_t)(ke - kb) * per_angle > ws->partial_floats) {
            set_error("forward workspace too small");
            return PT_EINVAL;
        }
        FwdArgs a;
        a.x = x;
        a.x2 = x2;
        a.partial = ws->partial;
        a.tab = plan->d_tab;
        a.sel_angle = sel->d_angle;
        a.bpos0 = sel->d_branch_pos[0];
        a.bpos1 = sel->d_branch_pos[1];
        int e0 = bi0, e1 = bi1;
        // the branch lists are ascending in selection slot: slice [kb, ke)
        {
            int c0 = 0, c1 = 0;
            for (int k = kb; k < ke; ++k) {
                if (plan->h_tab[sel->h_angle[k]].branch) ++c1; else ++c0;
            }
            e0 = bi0 + c0;
            e1 = bi1 + c1;
        }
        a.bbeg[0] = bi0; a.bend[0] = e0;
        a.bbeg[1] = bi1; a.bend[1] = e1;
        a.k_begin = kb;
        a.n_k = ke - kb;
        a.H = plan->H; a.W = plan->W; a.Z = plan->Z; a.B = plan->B;
        a.n_bands = n_bands;
        // angle groups: enough CTAs for >= ~4 waves of 2 CTAs/SM on big launches
        const int max_branch = std::max(e0 - bi0, e1 - bi1);
        const long long base_ctas = (long long)n_tiles * n_bands * plan->Z * 2;
        long long want = (long long)plan->sm_count * 2 * 4;
        int groups = (int)std::min<long long>(std::max(1LL, want / std::max(1LL, base_ctas)),
                                              std::max(1, (max_branch + 3) / 4));
        a.n_groups = std::max(1, groups);
        dim3 grid(n_tiles, n_bands * plan->Z, 2 * a.n_groups);
        {
            ProfScope ps(ws, PT_PROF_FWD_BAND, st);
            fwd_band_kernel<TY, TX, NT><<<grid, NT, T::SMEM, st>>>(a);
            PT_CHECK_LAUNCH();
        }

        RedArgs r;
        r.partial = ws->partial;
        r.tab = plan->d_tab;
        r.sel_angle = sel->d_angle;
        r.k_begin = kb;
        r.n_k = ke - kb;
        r.Z = plan->Z;
        r.B = plan->B;
        r.nb_row = nb_row;
        r.nb_col = nb_col;
        r.data = data;
        r.y = y;
        r.block_sums = sumsq ? ws->red + red_off : nullptr;
        const size_t tot = (size_t)(ke - kb) * plan->Z * plan->B;
        const int nblk = (int)((tot + 255) / 256);
        {
            ProfScope ps(ws, PT_PROF_FWD_REDUCE, st);
            fwd_reduce_kernel<<<nblk, 256, 0, st>>>(r);
            PT_CHECK_LAUNCH();
        }
        red_off += nblk;
        bi0 = e0;
        bi1 = e1;
    }
    if (sumsq) {
        return launch_sum_doubles(ws->red, red_off, sumsq, 0, st);
    }
    return PT_OK;
}

int launch_forward(pt_plan* plan, Workspace* ws, const pt_selection* sel, const float* x,
                   const float* x2, const float* data, float* y, double* sumsq, cudaStream_t st)
{
    if (sel->n == 0) {
        if (sumsq) PT_CHECK_CUDA(cudaMemsetAsync(sumsq, 0, sizeof(double), st));
        return PT_OK;
    }
    switch (plan->fwd_ty) {
        case 64: return run_forward_cfg<64, 256, 256>(plan, ws, sel, x, x2, data, y, sumsq, st);
        case 32: return run_forward_cfg<32, 128, 256>(plan, ws, sel, x, x2, data, y, sumsq, st);
        default: return run_forward_cfg<16, 64, 128>(plan, ws, sel, x, x2, data, y, sumsq, st);
    }
}

// ---------------------------------------------------------------------------
// Adjoint: pixel-driven gather.  For pixel (r, c) and one angle, the rays
// whose Joseph taps land on it are those with |pos_b - lane| < 1 at its step,
// i.e. bins b near the crossing b_f = (lane - pos_0)/sigma; the weight is the
// hat function step_len * max(0, 1 - |pos_b - lane|), which equals the
// reference's (1-frac) / frac taps (projector.py:49-60).  With bin spacing >=
// pixel size (|sigma| >= 1) exactly the two bins floor(b_f), floor(b_f)+1 can
// contribute ("two-tap"); otherwise 2*ceil(1/|sigma|) candidates are scanned.
// One CTA = TR x TC pixels; a chunk of NA angles has its parameters (in the
// tile frame, float64 -> float32) and the sinogram bins it touches (scaled by
// step_len) staged in shared memory, then every thread accumulates its 8
// pixels over the chunk.  Sums are two-level (per chunk, then across chunks).
// ---------------------------------------------------------------------------
struct AdjArgs {
    const float* y;
    const AngleTab* tab;
    const int32_t* sel_angle;
    int32_t n_sel;
    int32_t H, W, Z, B;
    int32_t slot;
    int32_t cand_half;
    float alpha;
    int32_t accumulate;
    float* out;
    int32_t mode;  // 0 plain adjoint, 1 fused step epilogue
    pt_step_epilogue ep;
};

__device__ __forceinline__ void step_epilogue(const pt_step_epilogue& ep, size_t p, float g)
{
    float est;
    switch (ep.estimator) {
        case PT_EST_FULL: est = g; break;
        case PT_EST_SGD: est = ep.n_scale * g; break;
        case PT_EST_SAGA: {
            const float old = ep.aux0[p];
            const float s = ep.aux1[p];
            est = ep.n_scale * g + (s - ep.n_scale * old);
            ep.aux1[p] = (s - old) + g;
            ep.aux0[p] = g;
            break;
        }
        default: est = ep.n_scale * g + ep.aux0[p]; break;  // svrg / lsvrg
    }
    const float hv = ep.h[p];
    const float base = ep.x[p] - ep.gamma * est;
    const float xh = base + ep.gamma * hv;
    if (ep.theta) {
        ep.v_out[p] = base + ep.hcoef * hv;
        ep.xhat_out[p] = xh;
    } else {
        ep.x_out[p] = xh;
        if (!isfinite(xh) && ep.bad_iter)
            atomicMin((long long*)ep.bad_iter, (long long)ep.iteration);
    }
}

template <int TR, int TC, int NT, int NA, bool TWO_TAP>
__global__ void __launch_bounds__(NT) adj_gather_kernel(AdjArgs P)
{
    constexpr int PIX = TR * TC / NT;  // pixels per thread
    constexpr int ROWSTEP = NT / TC;
    extern __shared__ float slots[];
    __shared__ float s_br[NA], s_bc[NA], s_e0[NA], s_sg[NA];
    __shared__ int s_off[NA];

    const int tid = threadIdx.x;
    const int cl = tid % TC;
    const int rg = tid / TC;
    const int r0 = blockIdx.y * TR;
    const int c0 = blockIdx.x * TC;
    const int z = blockIdx.z;
    const size_t plane = (size_t)P.H * P.W;

    float acc_o[PIX];
#pragma unroll
    for (int j = 0; j < PIX; ++j) acc_o[j] = 0.f;

    for (int kb = 0; kb < P.n_sel; kb += NA) {
        const int nc = min(NA, P.n_sel - kb);
        if (tid < nc) {
            const int k = kb + tid;
            const AngleTab t = P.tab[P.sel_angle[k]];
            // d(b, r, c) = sigma*b + ar*r + ac*c + a0
            const double ar = t.branch ? -1.0 : t.m;
            const double ac = t.branch ? t.m : -1.0;
            const double bf00 = -(ar * r0 + ac * c0 + t.a0) / t.sigma;
            const double bref = floor(bf00);
            const double br = -ar / t.sigma, bc = -ac / t.sigma;
            const double e0 = bf00 - bref;
            // local crossing range over the tile corners
            const double v1 = e0 + br * (TR - 1), v2 = e0 + bc * (TC - 1);
            const double v3 = e0 + br * (TR - 1) + bc * (TC - 1);
            const double lo = fmin(fmin(e0, v1), fmin(v2, v3));
            const int jlo = (int)floor(lo) - P.cand_half - 1;
            s_br[tid] = (float)br;
            s_bc[tid] = (float)bc;
            s_e0[tid] = (float)e0;
            s_sg[tid] = (float)fabs(t.sigma);
            s_off[tid] = -jlo;  // slot index of local bin 0
            // global bin of slot index 0 stored in the slot header region below
            reinterpret_cast<int*>(slots)[tid] = (int)bref + jlo;
        }
        __syncthreads();
        // stage the touched bins (scaled by step_len), zero outside [0, B)
        float* sl = slots + NA;
        for (int idx = tid; idx < nc * P.slot; idx += NT) {
            const int a = idx / P.slot, j = idx - a * P.slot;
            const int k = kb + a;
            const int b = reinterpret_cast<const int*>(slots)[a] + j;
            float v = 0.f;
            if (b >= 0 && b < P.B) {
                const AngleTab t = P.tab[P.sel_angle[k]];
                v = P.y[((size_t)k * P.Z + z) * P.B + b] * t.step_len;
            }
            sl[idx] = v;
        }
        __syncthreads();
        float acc_i[PIX];
#pragma unroll
        for (int j = 0; j < PIX; ++j) acc_i[j] = 0.f;
        for (int a = 0; a < nc; ++a) {
            const float br = s_br[a], sg = s_sg[a];
            const float cterm = fmaf((float)cl, s_bc[a], s_e0[a]);
            const int ybase = a * P.slot + s_off[a] - kMagicBits;
#pragma unroll
            for (int j = 0; j < PIX; ++j) {
                const float bl = fmaf((float)(rg + j * ROWSTEP), br, cterm);
                const float tt = __fadd_rd(bl, kMagic);
                const float phi = bl - (tt - kMagic);
                const float* yp = sl + (ybase + __float_as_int(tt));
                if (TWO_TAP) {
                    const float w0 = fmaxf(0.f, fmaf(-sg, phi, 1.f));
                    const float w1 = fmaxf(0.f, fmaf(sg, phi, 1.f - sg));
                    acc_i[j] = fmaf(w0, yp[0], fmaf(w1, yp[1], acc_i[j]));
                } else {
                    for (int q = -P.cand_half + 1; q <= P.cand_half; ++q) {
                        const float w = fmaxf(0.f, 1.f - sg * fabsf((float)q - phi));
                        acc_i[j] = fmaf(w, yp[q], acc_i[j]);
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < PIX; ++j) acc_o[j] += acc_i[j];
        __syncthreads();
    }

    const int c = c0 + cl;
    if (c >= P.W) return;
#pragma unroll
    for (int j = 0; j < PIX; ++j) {
        const int r = r0 + rg + j * ROWSTEP;
        if (r >= P.H) continue;
        const size_t p = (size_t)z * plane + (size_t)r * P.W + c;
        if (P.mode == 0) {
            float v = P.alpha * acc_o[j];
            if (P.accumulate) v += P.out[p];
            P.out[p] = v;
        } else {
            step_epilogue(P.ep, p, acc_o[j]);
        }
    }
}

__global__ void epilogue_kernel(const float* g, size_t n, pt_step_epilogue ep)
{
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (size_t)gridDim.x * blockDim.x)
        step_epilogue(ep, p, g[p]);
}

static constexpr int kTR = 32, kTC = 64, kNT = 256, kNA = 32;

template <bool TWO>
static int run_gather(pt_plan* plan, const AdjArgs& a, cudaStream_t st)
{
    const size_t smem = (size_t)(kNA + kNA * a.slot) * sizeof(float);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        PT_CHECK_CUDA(cudaFuncSetAttribute(adj_gather_kernel<kTR, kTC, kNT, kNA, TWO>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        attr = smem;
    }
    dim3 grid((plan->W + kTC - 1) / kTC, (plan->H + kTR - 1) / kTR, plan->Z);
    adj_gather_kernel<kTR, kTC, kNT, kNA, TWO><<<grid, kNT, smem, st>>>(a);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

int launch_adjoint(pt_plan* plan, const pt_selection* sel, const float* y, float* x_out,
                   float alpha, int accumulate, const pt_step_epilogue* ep, cudaStream_t st,
                   Workspace* ws, int cat)
{
    ProfScope ps(ws, cat, st);
    AdjArgs a;
    a.y = y;
    a.tab = plan->d_tab;
    a.sel_angle = sel->d_angle;
    a.n_sel = sel->n;
    a.H = plan->H; a.W = plan->W; a.Z = plan->Z; a.B = plan->B;
    a.slot = plan->gather_slot;
    a.cand_half = plan->cand_half;
    a.alpha = alpha;
    a.accumulate = accumulate;
    a.out = x_out;
    a.mode = ep ? 1 : 0;
    if (ep) a.ep = *ep; else memset(&a.ep, 0, sizeof(a.ep));
    if (plan->cand_half == 1) return run_gather<true>(plan, a, st);
    return run_gather<false>(plan, a, st);
}

int launch_epilogue(pt_plan* plan, const float* g, const pt_step_epilogue* ep, cudaStream_t st)
{
    const size_t n = (size_t)plan->Z * plan->H * plan->W;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)plan->sm_count * 8);
    epilogue_kernel<<<blocks, 256, 0, st>>>(g, n, *ep);
    PT_CHECK_LAUNCH();
    return PT_OK;
}

}  // namespace pt
