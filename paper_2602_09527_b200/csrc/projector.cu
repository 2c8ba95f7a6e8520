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
#include <cstdlib>
#include <cstring>

#include "pt_internal.cuh"
#include "pt_simd.cuh"
#include "pt_joseph.cuh"

namespace pt {

// ---------------------------------------------------------------------------
// Forward: a work item = one band of TY consecutive steps (image rows for
// row-stepping angles, image columns for column-stepping ones) x one tile of
// TX lanes (+ halo), for one group of the selection's angles of that branch.
// One CTA per item; its tile is staged in shared memory by cp.async (LDGSTS,
// zero-filled outside the image) while warp 0 builds the first chunk's ray
// tables, and co-resident CTAs overlap one another's staging.  Both
// branches keep the image's row-major orientation in shared memory (the
// column branch reads lanes with an odd pitch -> conflict-free).  For each ray
// it owns (ray position at the band's middle step inside [l0, l0+TX); the edge
// tiles also own the rays beyond), a thread sums the <= TY Joseph samples of
// that ray inside the band.  Each (band, ray) partial is written exactly once,
// so the band reduction that follows is deterministic and needs no atomics.
// Partial sums of <= 64 samples are combined in float64.
// ---------------------------------------------------------------------------
// Forward tile configurations: (id, band height TY, lane tile TX, threads, min CTAs/SM)
#define PT_FWD_CONFIGS(X)        \
    X(0, 64, 256, 256, 2)        \
    X(1, 64, 128, 256, 4)        \
    X(2, 32, 256, 256, 4)        \
    X(3, 64, 256, 512, 2)        \
    X(4, 32, 512, 256, 3)        \
    X(5, 16, 256, 256, 4)        \
    X(6, 32, 256, 128, 8)        \
    X(7, 32, 128, 128, 8)        \
    X(100, 32, 128, 256, 4)      \
    X(101, 16, 64, 128, 8)

void forward_config(int cfg, int32_t* ty, int32_t* tx)
{
    switch (cfg) {
#define PT_FWD_TT(id, TY, TX, NT, MB) \
    case id: *ty = TY; *tx = TX; return;
        PT_FWD_CONFIGS(PT_FWD_TT)
#undef PT_FWD_TT
        default: *ty = 32; *tx = 256; return;
    }
}

struct FwdArgs {
    int tma;  // row-branch tiles by TMA (W % 4 == 0, 16-byte aligned image)
    const float* x;
    float* partial;
    const AngleTab* tab;
    const int32_t* sel_angle;
    const int32_t* bpos0;
    const int32_t* bpos1;
    int32_t bbeg[2], bend[2];
    int32_t k_begin, n_k;
    int32_t H, W, Z, B;
    int32_t n_groups;
    int32_t n_bands;  // bands per slice (max over branches)
    int32_t n_tiles;  // lane tiles (max over branches)
};

template <int TY, int TX>
struct FwdTile {
    static constexpr int HL = ((TY / 2 + 3) + 3) & ~3;     // halo, a multiple of 4 lanes
    static constexpr int NL = TX + 2 * HL;                 // lanes staged per band
    static constexpr int PITCH_R = NL;                      // row branch: [TY][NL] (the TMA box)
    static constexpr int PITCH_C = TY + 1;                  // column branch: [NL][PITCH_C]
    static constexpr int BUF = (TY * PITCH_R > NL * PITCH_C) ? TY * PITCH_R : NL * PITCH_C;
    static constexpr int SMEM = BUF * 4;
};

struct FwdItem {
    int z, branch, band, tile, group;
};

// grid = (tile, band + n_bands * group, branch + 2 * z): one runtime division
__device__ __forceinline__ FwdItem decode_item(const FwdArgs& P)
{
    FwdItem it;
    it.tile = blockIdx.x;
    it.group = blockIdx.y / (unsigned)P.n_bands;
    it.band = blockIdx.y - it.group * P.n_bands;
    it.branch = blockIdx.z & 1;
    it.z = blockIdx.z >> 1;
    return it;
}

// [lo, hi) of the group's angles within the branch list (nb * n_groups < 2^31
// is checked on the host)
__device__ __forceinline__ int group_begin(int nb, int group, int n_groups)
{
    return (int)((unsigned)(nb * group) / (unsigned)n_groups);
}

// true when the item has work (band / tile inside the branch's extent, angles in the group)
__device__ __forceinline__ bool item_valid(const FwdArgs& P, const FwdItem& it, int TY, int TX)
{
    const int n_steps = it.branch ? P.W : P.H;
    const int n_lanes = it.branch ? P.H : P.W;
    if (it.band * TY >= n_steps || it.tile * TX >= n_lanes) return false;
    const int nb = it.branch ? P.bend[1] - P.bbeg[1] : P.bend[0] - P.bbeg[0];
    return group_begin(nb, it.group + 1, P.n_groups) > group_begin(nb, it.group, P.n_groups);
}

// Threads [t0, t0 + nthr) (whole warps) copy the tile.
template <int TY, int TX, int NT>
__device__ __forceinline__ void stage_tile(const FwdArgs& P, const FwdItem& it, uint32_t buf,
                                           int t0, int nthr)
{
    using T = FwdTile<TY, TX>;
    const int NW = nthr >> 5;
    const int warp = (threadIdx.x - t0) >> 5, lane = threadIdx.x & 31;
    const int s0 = it.band * TY;
    const int lane_org = it.tile * TX - T::HL;
    const float* img = P.x + (size_t)it.z * P.H * P.W;
    const int n_steps = it.branch ? P.W : P.H;
    const int n_lanes = it.branch ? P.H : P.W;
    if (s0 + TY <= n_steps && lane_org >= 0 && lane_org + T::NL <= n_lanes &&
        (it.branch == 1 || (P.W & 3) == 0)) {
        // interior tile (the common case): no bounds tests, one 64-bit base,
        // 32-bit offsets, a warp per staged row
        if (it.branch == 0) {
            // [st][ll] = img[s0 + st][lane_org + ll], 16-byte copies
            constexpr int NQ = T::NL / 4;
            const float* src0 = img + ((size_t)s0 * P.W + lane_org);
            for (int st = warp; st < TY; st += NW) {
                const uint32_t so = (uint32_t)(st * P.W);
                const uint32_t dst = buf + (uint32_t)(st * T::PITCH_R) * 4u;
#pragma unroll
                for (int u = 0; u < (NQ + 31) / 32; ++u) {
                    const int q = lane + 32 * u;
                    if (NQ % 32 == 0 || q < NQ) cp_async16(dst + 16u * q, src0 + (so + 4u * q), 16);
                }
            }
        } else {
            // [ll][st] = img[lane_org + ll][s0 + st], 4-byte copies into the odd pitch
            const float* src0 = img + ((size_t)lane_org * P.W + s0);
            for (int ll = warp; ll < T::NL; ll += NW) {
                const uint32_t so = (uint32_t)(ll * P.W) + lane;
                const uint32_t dst = buf + (uint32_t)(ll * T::PITCH_C + lane) * 4u;
#pragma unroll
                for (int u = 0; u < (TY + 31) / 32; ++u) {
                    if (TY % 32 != 0 && lane + 32 * u >= TY) break;
                    cp_async4(dst + 128u * u, src0 + (so + 32u * u), true);
                }
            }
        }
        return;
    }
    if (it.branch == 0 && (P.W & 3) == 0) {
        // [st][ll] = img[s0 + st][lane_org + ll]: 16-byte copies (lane_org and
        // W are multiples of 4), zero-filled outside the image
        constexpr int NQ = T::NL / 4;
        const int i0 = threadIdx.x - t0;
        int st = i0 / NQ, qq = i0 - st * NQ;
        const int dst_ = nthr / NQ, dq = nthr - dst_ * NQ;
        while (st < TY) {
            const int r = s0 + st, c = lane_org + 4 * qq;
            const bool ok = r < P.H && c >= 0 && c < P.W;  // whole 4-lane chunks
            cp_async16(buf + (uint32_t)(st * T::PITCH_R + 4 * qq) * 4u,
                       img + (ok ? r * P.W + c : 0), ok ? 16 : 0);
            st += dst_;
            qq += dq;
            if (qq >= NQ) { qq -= NQ; ++st; }
        }
    } else if (it.branch == 0) {
        // [st][ll] = img[s0 + st][lane_org + ll]: a warp per tile row
        for (int st = warp; st < TY; st += NW) {
            const int r = s0 + st;
            const bool rin = r < P.H;
            const float* src = img + (size_t)(rin ? r : 0) * P.W;
            const uint32_t dst = buf + (uint32_t)(st * T::PITCH_R) * 4u;
#pragma unroll 4
            for (int ll = lane; ll < T::NL; ll += 32) {
                const int c = lane_org + ll;
                const bool ok = rin && c >= 0 && c < P.W;
                cp_async4(dst + (uint32_t)ll * 4u, src + (ok ? c : 0), ok);
            }
        }
    } else {
        // [ll][st] = img[lane_org + ll][s0 + st]: a warp per image-row segment
        const int nst = min(TY, P.W - s0);  // steps inside the image
        const int r_lo = max(0, -lane_org), r_hi = min(T::NL, P.H - lane_org);
        for (int ll = warp; ll < T::NL; ll += NW) {
            const bool rin = ll >= r_lo && ll < r_hi;
            const float* src = img + (rin ? (lane_org + ll) * P.W + s0 : 0);
            const uint32_t dst = buf + (uint32_t)(ll * T::PITCH_C + lane) * 4u;
#pragma unroll
            for (int u = 0; u < (TY + 31) / 32; ++u) {
                if (TY % 32 != 0 && lane + 32 * u >= TY) break;
                const bool ok = rin && lane + 32 * u < nst;
                cp_async4(dst + 128u * u, src + (ok ? lane + 32 * u : 0), ok);
            }
        }
    }
}

// Row-branch tile by TMA: the image as a 4D tensor (4, W/4, H, Z) and one box
// (4, NL/4, TY, 1) lands as the dense [TY][NL] tile; coordinates outside the
// image (negative lane origin, the last band, the last tile) are zero-filled
// by the copy engine, which is exactly the reference's "rays outside the grid
// contribute 0".  One elected thread issues it; completion on an mbarrier.
__device__ __forceinline__ void fwd_tma_issue(const CUtensorMap* map, uint32_t dst, uint32_t bar,
                                              int lane_org, int s0, int z, uint32_t bytes)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes));
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(map), "r"(0), "r"(lane_org >> 2), "r"(s0), "r"(z), "r"(bar) : "memory");
}
__device__ __forceinline__ void fwd_mbar_wait(uint32_t bar)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "FW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra FW_%=;\n}" ::"r"(bar));
}

template <int TY, int TX, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) fwd_band_kernel(FwdArgs P,
                                                            const __grid_constant__ CUtensorMap tmap)
{
    using T = FwdTile<TY, TX>;
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t s_bar;
    constexpr int CH = 32;
    __shared__ int s_pref[CH + 1];
    __shared__ int2 s_bk[CH];       // {first owned ray, selection slot}
    __shared__ float4 s_ray[CH];    // {tile-local lane of ray blo at st 0, sigma, m, 1/m}
    __shared__ float* s_out[CH];    // partial of ray blo in this band

    const int tid = threadIdx.x;
    const FwdItem it = decode_item(P);
    if (!item_valid(P, it, TY, TX)) return;
    const uint32_t tile_u32 = smem_u32(sm);
    // warp 0 builds the first chunk's ray tables (static data) while the
    // predecessor drains; the other warps wait for it and stage the image tile
    const bool stager = tid >= 32;
    const bool tma = P.tma && it.branch == 0;
    const uint32_t bar = smem_u32(&s_bar);
    if (stager) {
        pdl_wait<PDL_FWD>();  // the image is the predecessor's output
        if (tma) {
            if (tid == 32)
                fwd_tma_issue(&tmap, tile_u32, bar, it.tile * TX - T::HL, it.band * TY, it.z,
                              (uint32_t)(TY * T::NL * 4));
        } else {
            stage_tile<TY, TX, NT>(P, it, tile_u32, 32, NT - 32);
            cp_async_commit();
        }
    }

    const int branch = it.branch;
    const int n_steps = branch ? P.W : P.H;
    const int n_lanes = branch ? P.H : P.W;
    const int s0 = it.band * TY;
    const int l0 = it.tile * TX;
    const int lane_org = l0 - T::HL;
    const int ty_valid = min(TY, n_steps - s0);
    const int bb = branch ? P.bbeg[1] : P.bbeg[0];
    const int nb = (branch ? P.bend[1] : P.bend[0]) - bb;
    const int a_begin = bb + group_begin(nb, it.group, P.n_groups);
    const int a_end = bb + group_begin(nb, it.group + 1, P.n_groups);
    const int32_t* bpos = branch ? P.bpos1 : P.bpos0;
    const bool first_tile = (l0 == 0);
    const bool last_tile = (l0 + TX >= n_lanes);
    // owned rays drift at most TY/2 lanes (|m| <= 1) from their band-middle
    // position in [l0, l0 + TX): away from the image edges no ray leaves the
    // image inside the band, so the per-ray step clipping is skipped
    const bool interior = !first_tile && !last_tile && l0 >= TY / 2 + 2 &&
                          l0 + TX + TY / 2 + 2 <= n_lanes;
    const double smid = s0 + 0.5 * (ty_valid - 1);
    bool waited = false;

    for (int cbeg = a_begin; cbeg < a_end; cbeg += CH) {
        const int nc = min(CH, a_end - cbeg);
        // per-angle ray ranges (overlaps the tile copy on the first chunk)
        if (tid < CH) {
            int cnt = 0;
            if (tid < nc) {
                const int k = bpos[cbeg + tid];
                const AngleTab t = P.tab[P.sel_angle[k]];
                // rays owned by this tile: pos at the middle step in [lo, hi)
                const double base = t.a0 + smid * t.m;
                long long blo, bhi;
                if (t.sigma > 0) {
                    blo = first_tile ? 0 : (long long)ceil(((double)l0 - base) * t.isig);
                    bhi = last_tile ? P.B : (long long)ceil(((double)(l0 + TX) - base) * t.isig);
                } else {
                    blo = last_tile ? 0 : (long long)floor(((double)(l0 + TX) - base) * t.isig) + 1;
                    bhi = first_tile ? P.B : (long long)floor(((double)l0 - base) * t.isig) + 1;
                }
                blo = max(blo, 0LL);
                bhi = min(bhi, (long long)P.B);
                cnt = (int)max(0LL, bhi - blo);
                s_bk[tid] = make_int2((int)blo, k);
                s_out[tid] = P.partial +
                             ((((size_t)it.band * P.n_k + (size_t)(k - P.k_begin)) * P.Z + it.z) *
                                  P.B + (size_t)blo);
                // tile-local lane position of ray blo at step 0 (float64 -> float32;
                // per ray only (b - blo) * sigma, |.| <~ TX, is added in float32)
                s_ray[tid] = make_float4(
                    (float)(t.a0 + (double)blo * t.sigma + (double)s0 * t.m - (double)lane_org),
                    (float)t.sigma, (float)t.m, (float)t.im);
            }
            int v = cnt;  // inclusive warp scan of the ray counts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int n = __shfl_up_sync(0xffffffffu, v, o);
                if (tid >= o) v += n;
            }
            s_pref[tid + 1] = v;
            if (tid == 0) s_pref[0] = 0;
        }
        if (!waited) {
            if (!stager) pdl_wait<PDL_FWD>();
            else if (!tma) cp_async_wait_all();
        }
        __syncthreads();
        if (!waited) {
            if (tma) fwd_mbar_wait(bar);  // after the barrier: the mbarrier is initialised
            waited = true;
        }
        const int total = s_pref[nc];
        int j = 0;
        for (int w = tid; w < total; w += NT) {
            while (w >= s_pref[j + 1]) ++j;
            const int db = w - s_pref[j];
            const float4 ry = s_ray[j];
            const float mf = ry.z;
            const float pl = fmaf((float)db, ry.y, ry.x);  // tile-local lane at st = 0
            // steps where pos in [-1.5, n_lanes + 0.5] (global lanes): outside,
            // both taps are zero (float32 is ample for a 0.5-lane margin)
            const float P0 = pl + (float)lane_org;
            int st_a = 0, st_b = ty_valid;
            const float im = ry.w;
            if (interior) {
            } else if (im == 0.f) {
                if (P0 < -1.5f || P0 > n_lanes + 0.5f) st_b = 0;
            } else {
                const float e1 = (-1.5f - P0) * im, e2 = ((float)n_lanes + 0.5f - P0) * im;
                const float lo = fminf(e1, e2), hi = fmaxf(e1, e2);
                st_a = max(st_a, (int)ceilf(fminf(fmaxf(lo, -1.f), (float)TY + 1.f)));
                st_b = min(st_b, (int)floorf(fminf(fmaxf(hi, -2.f), (float)TY + 1.f)) + 1);
            }
            const float acc = branch == 0
                ? ray_band_sum<4, T::PITCH_R * 4>(tile_u32, st_a, st_b, pl, mf)
                : ray_band_sum<T::PITCH_C * 4, 4>(tile_u32, st_a, st_b, pl, mf);
            s_out[j][db] = acc;
        }
        if (cbeg + CH < a_end) __syncthreads();  // chunk tables are rewritten next
    }
    pdl_trigger<PDL_FWD>();
}

__global__ void sub_images_kernel(const float* a, const float* b, float* out, size_t n)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = a[i] - b[i];
}

struct RedArgs {
    const float* partial;
    const AngleTab* tab;
    const int32_t* sel_angle;
    int32_t k_begin, n_k, Z, B;
    int32_t nb_row, nb_col;
    const float* data;
    const float* data2;
    float* y;
    double* block_sums;
    double* y64;  // row-slab partial: s * step_len in float64, no data, no y
};

__global__ void __launch_bounds__(256) fwd_reduce_kernel(RedArgs P)
{
    pdl_wait<PDL_REDUCE>();
    // n_k * Z * B < 2^31 (checked on the host): 32-bit index math
    const unsigned total = (unsigned)P.n_k * P.Z * P.B;
    const unsigned idx = blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (idx < total) {
        const unsigned t = idx / (unsigned)P.B;
        const int b = (int)(idx - t * P.B);
        const int kk = (int)(t / (unsigned)P.Z);
        const int z = (int)(t - kk * P.Z);
        const int k = kk + P.k_begin;
        const int ang = P.sel_angle[k];
        const AngleTab at = P.tab[ang];
        // square images: the band count does not depend on the branch, so the
        // partial loads need not wait for the angle-table load (latency chain)
        const int nb = (P.nb_row == P.nb_col) ? P.nb_row : at.branch ? P.nb_col : P.nb_row;
        const size_t stride = (size_t)P.n_k * P.Z * P.B;
        // four independent float64 partial sums (latency), combined pairwise
        const float* pp = P.partial + idx;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int band = 0;
        // 16 loads in flight before the first add (the partials sit in L2);
        // the same accumulator assignment and order as the 4-band loop below
        for (; band + 16 <= nb; band += 16) {
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = __ldcs(pp + (size_t)(band + i) * stride);
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
                s0 += v[i]; s1 += v[i + 1]; s2 += v[i + 2]; s3 += v[i + 3];
            }
        }
        for (; band + 4 <= nb; band += 4) {
            const float a = __ldcs(pp + (size_t)band * stride);
            const float b2 = __ldcs(pp + (size_t)(band + 1) * stride);
            const float c = __ldcs(pp + (size_t)(band + 2) * stride);
            const float d = __ldcs(pp + (size_t)(band + 3) * stride);
            s0 += a; s1 += b2; s2 += c; s3 += d;
        }
        for (; band < nb; ++band) s0 += __ldcs(pp + (size_t)band * stride);
        const double s = (s0 + s1) + (s2 + s3);
        double yd = s * (double)at.step_len;
        if (P.y64) {  // partial line integrals of a row slab (summed over ranks later)
            P.y64[((size_t)k * P.Z + z) * P.B + b] = yd;
            pdl_trigger<PDL_REDUCE>();
            return;
        }
        if (P.data) yd -= (double)P.data[((size_t)ang * P.Z + z) * P.B + b];
        if (P.data2) yd -= (double)P.data2[((size_t)ang * P.Z + z) * P.B + b];
        const float yv = (float)yd;
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
    pdl_trigger<PDL_REDUCE>();
}

// ---------------------------------------------------------------------------
// Small images (pt_joseph.cuh): one launch writes finished residual rows --
// no band partials, no reduction launch.  Every CTA stages the whole image
// (one TMA box into a dense [132][136] layout when W % 4 == 0, else cp.async
// into the odd-pitch [132][133] one; 4-byte cp.async of 70 KB per CTA took
// ~4 us, the box ~1.5 us) and sums 32 * RW consecutive rays of the selection, one warp per segment
// (lanes = adjacent rays); the segment sums are combined in float64 in
// segment order, then scaled, and the data rows subtracted, exactly as
// fwd_reduce_kernel does.  A ray's value does not depend on which CTA
// computes it, so subsets and the full selection agree bitwise (and the
// cluster-resident executor, cluster.cu, reproduces it bit for bit).
// ---------------------------------------------------------------------------
struct SmallArgs {
    const float* x;
    const AngleTab* tab;
    const int32_t* sel_angle;
    int32_t n_k, H, W, B;
    const float* data;
    const float* data2;
    float* y;
    double* block_sums;
    double* y64;  // row-slab partial: s * step_len in float64, no data, no y
};

template <int PITCH>
__global__ void __launch_bounds__(1024) fwd_small_kernel(SmallArgs a,
                                                         const __grid_constant__ CUtensorMap tmap)
{
    extern __shared__ __align__(128) float img[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ float part[kSmallNseg][64];
    __shared__ double red[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nw = blockDim.x >> 5;
    const int rw = warp / kSmallNseg, seg = warp - rw * kSmallNseg;
    const int rays_cta = 32 * (nw / kSmallNseg);
    const int rl = rw * 32 + lane;  // ray within the CTA
    const uint32_t buf = smem_u32(img);

    // ray tables first (static data: overlaps the predecessor's tail)
    const int total = a.n_k * a.B;
    const int ray = blockIdx.x * rays_cta + rl;
    const bool live = ray < total;
    const int k = live ? ray / a.B : 0;
    const int b = live ? ray - k * a.B : 0;
    const int ang = a.sel_angle[k];
    const AngleTab t = a.tab[ang];
    const SmallRay sr = small_ray(t, b, a.H, a.W);

    const uint32_t bar = smem_u32(&s_bar);
    if (PITCH == kSmallPitchT) {
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
        __syncthreads();  // the barrier is initialised before anyone waits on it
    }
    pdl_wait<PDL_FWD_SMALL>();  // the image is the predecessor's output
    if (PITCH == kSmallPitchT) {
        if (tid == 0) small_stage_tma(&tmap, buf, bar);
        small_mbar_wait(bar, 0);
    } else {
        small_stage(a.x, a.H, a.W, buf, 0, blockDim.x);
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
    }
    const float acc = live ? small_segment<PITCH>(buf, sr, seg) : 0.f;
    part[seg][rl] = acc;
    __syncthreads();
    double sq = 0.0;
    if (seg == 0 && live) {
        const double yd = small_line_integral(&part[0][rl], 64, t.step_len);
        const size_t o = (size_t)k * a.B + b;
        if (a.y64) {
            a.y64[o] = yd;
        } else {
            const float yv = residual_value(yd, a.data, a.data2, (size_t)ang * a.B + b);
            a.y[o] = yv;
            sq = (double)yv * (double)yv;
        }
    }
    if (a.block_sums) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, o);
        if (lane == 0) red[warp] = sq;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int i = 0; i < nw; ++i) s += red[i];
            a.block_sums[blockIdx.x] = s;
        }
    }
    pdl_trigger<PDL_FWD_SMALL>();
}

static bool forward_small_ok(const pt_plan* plan)
{
    static const bool on = [] {
        const char* e = getenv("PT_FWD_SMALL");
        return !(e && e[0] == '0');
    }();
    return on && plan->Z == 1 && plan->H <= kSmallMax && plan->W <= kSmallMax;
}

static int run_forward_small(pt_plan* plan, Workspace* ws, const pt_selection* sel,
                             const float* x, const float* data, float* y, double* sumsq,
                             cudaStream_t st, const float* data2, double* y64)
{
    // the whole image by one TMA box when its rows are 16-byte granular
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    const bool tma = (plan->W % 4) == 0 && (((uintptr_t)x & 15) == 0) && tma_available();
    if (tma) {
        const cuuint64_t dims[2] = {(cuuint64_t)plan->W, (cuuint64_t)plan->H};
        const cuuint32_t box[2] = {(cuuint32_t)kSmallPitchT, (cuuint32_t)kSmallRows};
        const int rc = make_map(&tmap, x, 2, dims, box);
        if (rc) return rc;
    }
    auto* kern = tma ? fwd_small_kernel<kSmallPitchT> : fwd_small_kernel<kSmallPitch>;
    {
        const int rc = ensure_smem((const void*)kern, kSmallSmem);
        if (rc) return rc;
    }
    const long long total = (long long)sel->n * plan->B;
    // rays per CTA: 32 (subsets: more CTAs) up to 128 (long selections: fewer
    // whole-image stagings)
    const long long per = total / (64LL * plan->sm_count);
    const int rw = (int)std::max(1LL, std::min(2LL, per));
    const int rays_cta = 32 * rw;
    const long long nblk = (total + rays_cta - 1) / rays_cta;
    if (nblk > INT32_MAX || (sumsq && (size_t)nblk > ws->red_doubles)) {
        set_error("forward launch too large");
        return PT_EINVAL;
    }
    SmallArgs a;
    a.x = x;
    a.tab = plan->d_tab;
    a.sel_angle = sel->d_angle;
    a.n_k = sel->n;
    a.H = plan->H;
    a.W = plan->W;
    a.B = plan->B;
    a.data = data;
    a.data2 = data2;
    a.y = y;
    a.block_sums = sumsq ? ws->red : nullptr;
    a.y64 = y64;
    {
        ProfScope ps(ws, PT_PROF_FWD_BAND, st);
        PT_CHECK_CUDA(launch_pdl(kern, dim3((unsigned)nblk), dim3(32 * kSmallNseg * rw),
                                 (size_t)kSmallSmem, st, a, tmap));
        PT_CHECK_LAUNCH();
    }
    if (sumsq) return launch_sum_doubles(ws->red, nblk, sumsq, 0, st);
    return PT_OK;
}

template <int TY, int TX, int NT, int MINB>
static int run_forward_cfg(pt_plan* plan, Workspace* ws, const pt_selection* sel,
                           const float* x, const float* x2, const float* data, float* y,
                           double* sumsq, cudaStream_t st, const float* data2, double* y64)
{
    using T = FwdTile<TY, TX>;
    {
        const int rc = ensure_smem((const void*)fwd_band_kernel<TY, TX, NT, MINB>, T::SMEM);
        if (rc) return rc;
    }
    if (x2) {
        // A (x - x2): difference image first (standalone API path; the solver
        // session never projects a difference, see session.cu)
        const size_t n = (size_t)plan->Z * plan->H * plan->W;
        if (ws->image_floats < n) { set_error("workspace image too small"); return PT_EINVAL; }
        sub_images_kernel<<<(int)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(
            x, x2, ws->image, n);
        PT_CHECK_LAUNCH();
        x = ws->image;
    }
    // row-branch tiles by TMA when the image rows are 16-byte granular
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    static const bool tma_env = [] {
        const char* e = getenv("PT_FWD_TMA");
        return !(e && e[0] == '0');
    }();
    int tma_ok = tma_env && (plan->W % 4 == 0) && (((uintptr_t)x & 15) == 0) && T::NL / 4 <= 256;
    if (tma_ok) {
        const cuuint64_t dims[4] = {4, (cuuint64_t)plan->W / 4, (cuuint64_t)plan->H,
                                    (cuuint64_t)plan->Z};
        const cuuint32_t box[4] = {4, (cuuint32_t)(T::NL / 4), (cuuint32_t)TY, 1};
        const int rc = make_map(&tmap, x, 4, dims, box);
        if (rc) return rc;
    }
    const int nb_row = (plan->H + TY - 1) / TY;
    const int nb_col = (plan->W + TY - 1) / TY;
    const int n_bands = plan->n_bands;
    const int n_tiles = (std::max(plan->H, plan->W) + TX - 1) / TX;
    const int n_chunk = std::max(1, plan->max_angles_per_launch);
    const size_t per_angle = (size_t)n_bands * plan->Z * plan->B;
    const int n_sel = sel->n;
    int n_blocks_red_total = 0;
    for (int kb = 0; kb < n_sel; kb += n_chunk) {
        int ke = std::min(n_sel, kb + n_chunk);
        n_blocks_red_total += (int)(((size_t)(ke - kb) * plan->Z * plan->B + 255) / 256);
    }
    if (sumsq && (size_t)n_blocks_red_total > ws->red_doubles) {
        set_error("reduction scratch too small");
        return PT_EINVAL;
    }
    static const int waves = [] {
        const char* e = getenv("PT_FWD_WAVES");
        return e ? std::max(1, atoi(e)) : 3;
    }();
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
        a.partial = ws->partial;
        a.tab = plan->d_tab;
        a.sel_angle = sel->d_angle;
        a.bpos0 = sel->d_branch_pos[0];
        a.bpos1 = sel->d_branch_pos[1];
        int c0 = 0, c1 = 0;  // the branch lists ascend in selection slot: slice [kb, ke)
        for (int k = kb; k < ke; ++k) {
            if (plan->h_tab[sel->h_angle[k]].branch) ++c1; else ++c0;
        }
        const int e0 = bi0 + c0, e1 = bi1 + c1;
        a.bbeg[0] = bi0; a.bend[0] = e0;
        a.bbeg[1] = bi1; a.bend[1] = e1;
        a.k_begin = kb;
        a.n_k = ke - kb;
        a.H = plan->H; a.W = plan->W; a.Z = plan->Z; a.B = plan->B;
        a.n_bands = n_bands;
        a.n_tiles = n_tiles;
        // one CTA per item; angle groups until ~`waves` waves of resident CTAs
        const int active_branches = (c0 > 0) + (c1 > 0);
        const long long base_items = (long long)n_tiles * n_bands * plan->Z * std::max(1, active_branches);
        const int max_branch = std::max(c0, c1);
        const long long slots = (long long)plan->sm_count * MINB;
        // long selections (the snapshot's 1800 angles) that fill few waves:
        // finer groups of >= ~56 angles balance the uneven items better
        // (config 2 full forward: 2 groups 3.42 ms, 8: 3.24, 16: 3.19, 32: 3.19)
        static const int groups_env = [] {
            const char* e = getenv("PT_FWD_GROUPS");
            return e ? std::max(1, atoi(e)) : 0;
        }();
        long long groups = (slots * waves + base_items - 1) / base_items;
        if (base_items < 8 * slots) groups = std::max<long long>(groups, std::min(16, max_branch / 56));
        if (groups_env) groups = groups_env;
        groups = std::max(1LL, std::min<long long>(groups, std::max(1, max_branch / 2)));
        a.n_groups = (int)groups;
        if ((long long)max_branch * (groups + 1) >= INT32_MAX ||
            (long long)n_bands * groups > 65535 || 2LL * plan->Z > 65535) {
            set_error("forward launch grid out of range");
            return PT_EINVAL;
        }
        const dim3 grid(n_tiles, (unsigned)(n_bands * groups), 2 * plan->Z);
        a.tma = tma_ok;
        {
            ProfScope ps(ws, PT_PROF_FWD_BAND, st);
            PT_CHECK_CUDA(launch_pdl(fwd_band_kernel<TY, TX, NT, MINB>, grid, dim3(NT),
                                     (size_t)T::SMEM, st, a, tmap));
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
        r.data2 = data2;
        r.y = y;
        r.block_sums = sumsq ? ws->red + red_off : nullptr;
        r.y64 = y64;
        const size_t tot = (size_t)(ke - kb) * plan->Z * plan->B;
        if (tot >= (size_t)INT32_MAX) {
            set_error("forward chunk too large for the band reduction");
            return PT_EINVAL;
        }
        const int nblk = (int)((tot + 255) / 256);
        {
            ProfScope ps(ws, PT_PROF_FWD_REDUCE, st);
            PT_CHECK_CUDA(launch_pdl(fwd_reduce_kernel, dim3(nblk), dim3(256), 0, st, r));
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
                   const float* x2, const float* data, float* y, double* sumsq, cudaStream_t st,
                   const float* data2, double* y64)
{
    if (sel->n == 0) {
        if (sumsq) PT_CHECK_CUDA(cudaMemsetAsync(sumsq, 0, sizeof(double), st));
        return PT_OK;
    }
    if (y64 && sumsq) { set_error("partial forward has no residual norm"); return PT_EINVAL; }
    if (forward_small_ok(plan)) {
        if (x2) {
            // A (x - x2): difference image first (standalone API path)
            const size_t n = (size_t)plan->H * plan->W;
            if (ws->image_floats < n) { set_error("workspace image too small"); return PT_EINVAL; }
            sub_images_kernel<<<(int)std::min<size_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(
                x, x2, ws->image, n);
            PT_CHECK_LAUNCH();
            x = ws->image;
        }
        return run_forward_small(plan, ws, sel, x, data, y, sumsq, st, data2, y64);
    }
    switch (plan->fwd_cfg) {
#define PT_FWD_CASE(id, TY, TX, NT, MB) \
    case id: return run_forward_cfg<TY, TX, NT, MB>(plan, ws, sel, x, x2, data, y, sumsq, st, data2, y64);
        PT_FWD_CONFIGS(PT_FWD_CASE)
#undef PT_FWD_CASE
        default: set_error("bad forward config"); return PT_EINVAL;
    }
}

// Row slabs: the summed float64 partial line integrals -> residual rows, with
// the reduction's own operation order (yd - data - data2, then float), so one
// slab reproduces the whole-image forward bit for bit.
__global__ void fwd_finish_kernel(const double* y64, const int32_t* sel_angle, int n_k, int Z,
                                  int B, const float* data, const float* data2, float* y)
{
    pdl_wait();
    const unsigned total = (unsigned)n_k * Z * B;
    for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += gridDim.x * blockDim.x) {
        const unsigned t = idx / (unsigned)B;
        const int b = (int)(idx - t * B);
        const int k = (int)(t / (unsigned)Z);
        const int z = (int)(t - k * Z);
        const int ang = sel_angle[k];
        double yd = y64[idx];
        if (data) yd -= (double)data[((size_t)ang * Z + z) * B + b];
        if (data2) yd -= (double)data2[((size_t)ang * Z + z) * B + b];
        y[idx] = (float)yd;
    }
    pdl_trigger();
}

int launch_forward_finish(pt_plan* plan, const pt_selection* sel, const double* y64,
                          const float* data, const float* data2, float* y, cudaStream_t st)
{
    if (sel->n == 0) return PT_OK;
    const size_t tot = (size_t)sel->n * plan->Z * plan->B;
    if (tot >= (size_t)INT32_MAX) { set_error("selection too large"); return PT_EINVAL; }
    const int blocks = (int)std::min<size_t>((tot + 255) / 256, (size_t)plan->sm_count * 8);
    PT_CHECK_CUDA(launch_pdl(fwd_finish_kernel, dim3(blocks), dim3(256), 0, st, y64,
                             (const int32_t*)sel->d_angle, sel->n, plan->Z, plan->B, data, data2,
                             y));
    PT_CHECK_LAUNCH();
    return PT_OK;
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
    int32_t vec;      // 16-byte staging: rows start at 4-aligned bins (B % 4 == 0, y 16B-aligned)
    int32_t cand_half;
    int32_t nbuf;     // staging buffers (2: chunk pipeline)
    int32_t n_epi;    // epilogue operand planes prefetched into shared memory
    float alpha;
    int32_t accumulate;
    float* out;
    int32_t mode;  // 0 plain adjoint, 1 fused step epilogue
    pt_step_epilogue ep;
    // plain adjoint split over angle parts (small images, long selections):
    // grid.z = Z * n_parts, part p sums angle chunks [p cpp, (p+1) cpp) into
    // out + p * Z * H * W; a combine kernel adds the parts in order
    int32_t n_parts, chunks_per_part;
};

// The estimator + ProxSkip step of one pixel (estimators.py:55,92-94,146;
// solvers.py:236-246) given its gradient g and the prefetched operands.
__device__ __forceinline__ void step_epilogue_vals(const pt_step_epilogue& ep, size_t p, float g,
                                                   float xv, float hv, float a0v, float a1v)
{
    float est;
    switch (ep.estimator) {
        case PT_EST_FULL: est = g; break;
        case PT_EST_SGD: est = ep.n_scale * g; break;
        case PT_EST_SAGA: {
            est = ep.n_scale * g + (a1v - ep.n_scale * a0v);
            ep.aux1[p] = (a1v - a0v) + g;
            ep.aux0[p] = g;
            break;
        }
        default: est = ep.n_scale * g + a0v; break;  // svrg / lsvrg
    }
    const float base = xv - ep.gamma * est;
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

__device__ __forceinline__ void step_epilogue(const pt_step_epilogue& ep, size_t p, float g)
{
    const bool saga = ep.estimator == PT_EST_SAGA;
    const bool vr = ep.estimator == PT_EST_SVRG || ep.estimator == PT_EST_LSVRG;
    step_epilogue_vals(ep, p, g, ep.x[p], ep.h[p], (saga || vr) ? ep.aux0[p] : 0.f,
                       saga ? ep.aux1[p] : 0.f);
}

template <int TR, int TC, int NT, int NA, bool TWO_TAP, int EPI>
__global__ void __launch_bounds__(NT, (TR * TC / NT > 8) ? 3 : 4) adj_gather_kernel(AdjArgs P0)
{
    // this CTA's angle part (P0.n_parts == 1: the whole selection)
    AdjArgs P = P0;
    const int part = (int)blockIdx.z / P0.Z;
    if (P0.n_parts > 1) {
        const int s0 = part * P0.chunks_per_part * NA;
        P.sel_angle = P0.sel_angle + s0;
        P.y = P0.y + (size_t)s0 * P0.Z * P0.B;
        P.n_sel = max(0, min(P0.n_sel - s0, P0.chunks_per_part * NA));
        P.out = P0.out + (size_t)part * P0.Z * P0.H * P0.W;
    }
    constexpr int PIX = TR * TC / NT;  // pixels per thread
    constexpr int NEPI = epi_planes(EPI);
    constexpr int ROWSTEP = NT / TC;
    constexpr int NW = NT / 32;
    extern __shared__ float smem[];
    // per-angle tile-frame parameters: {gbr, gbc, e0, S1} and {A0, y address}
    __shared__ float4 s_p4[2][NA];
    __shared__ float2 s_p2[2][NA];
    __shared__ int s_off[2][NA];
    __shared__ int s_bb[2][NA];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int cl = tid % TC;
    const int rg = tid / TC;
    const int r0 = blockIdx.y * TR;
    const int c0 = blockIdx.x * TC;
    const int z = (int)blockIdx.z - part * P0.Z;
    const size_t plane = (size_t)P.H * P.W;
    const uint32_t stage_u32 = smem_u32(smem);
    const uint32_t epi_u32 = stage_u32 + (uint32_t)(P.nbuf * NA * P.slot) * 4u;

    // --- epilogue operands: prefetched with cp.async, consumed at the end ---
    if (NEPI) {
        const bool vec = (P.W % 4) == 0;  // 16-byte rows (c0 is a multiple of TC)
        constexpr int Q = TC / 4;          // 16-byte quads per tile row
        static_assert(NT % Q == 0, "epilogue prefetch shape");
        constexpr int KQ = (TR * Q + NT - 1) / NT;  // copies per thread and plane
        if (vec && r0 + TR <= P.H && c0 + TC <= P.W) {
            // whole tile inside the image: one 64-bit base per plane, 32-bit
            // offsets stepping NT / Q rows per copy
            const int rl0 = tid / Q, q = tid % Q;
            const uint32_t off0 = (uint32_t)((r0 + rl0) * P.W + c0 + 4 * q);
            const uint32_t dst0 = epi_u32 + (uint32_t)(rl0 * TC + 4 * q) * 4u;
            const uint32_t dstep = (uint32_t)(NT / Q) * P.W;
#pragma unroll
            for (int e = 0; e < NEPI; ++e) {
                const float* srcp = e == 0 ? P.ep.x : e == 1 ? P.ep.h : e == 2 ? P.ep.aux0 : P.ep.aux1;
                const float* base = srcp + (size_t)z * plane;
#pragma unroll
                for (int k = 0; k < KQ; ++k) {
                    if ((TR * Q) % NT != 0 && rl0 + k * (NT / Q) >= TR) continue;
                    cp_async16(dst0 + (uint32_t)(e * TR * TC + k * (NT / Q) * TC) * 4u,
                               base + (off0 + (uint32_t)k * dstep), 16);
                }
            }
        } else for (int e = 0; e < NEPI; ++e) {
            const float* srcp = e == 0 ? P.ep.x : e == 1 ? P.ep.h : e == 2 ? P.ep.aux0 : P.ep.aux1;
            const float* base = srcp + (size_t)z * plane;
            const uint32_t dst = epi_u32 + (uint32_t)(e * TR * TC) * 4u;
            if (vec) {
                for (int idx = tid; idx < TR * Q; idx += NT) {
                    const int rl = idx / Q, q = idx - rl * Q;
                    const int r = r0 + rl, c = c0 + 4 * q;
                    const int nvalid = (r < P.H) ? max(0, min(4, P.W - c)) : 0;
                    cp_async16(dst + (uint32_t)(rl * TC + 4 * q) * 4u,
                               base + (nvalid ? (size_t)r * P.W + c : 0), 4 * nvalid);
                }
            } else {
                for (int idx = tid; idx < TR * TC; idx += NT) {
                    const int rl = idx / TC, cc = idx - rl * TC;
                    const int r = r0 + rl, c = c0 + cc;
                    const bool ok = r < P.H && c < P.W;
                    cp_async4(dst + (uint32_t)idx * 4u, base + (ok ? (size_t)r * P.W + c : 0), ok);
                }
            }
        }
        cp_async_commit();
    }

    // per-chunk preparation: angle parameters in the tile frame (float64 ->
    // float32) and the touched sinogram bins (cp.async, zero outside [0, B))
    // per-chunk preparation, split so the chunk's tile-frame parameters
    // (static data) can be formed before the PDL wait and only the staging of
    // the residual bins (the predecessor's output) after it.  One warp per
    // angle: every lane evaluates the parameters (float64 -> float32,
    // identical across lanes), lane 0 publishes them, the same warp's lanes
    // later stage the touched bins -- no CTA barrier.
    auto prepare_params = [&](int kb, int buf) {
        const int nc = min(NA, P.n_sel - kb);
        for (int a = warp; a < nc; a += NW) {
            const AngleTab& t = P.tab[P.sel_angle[kb + a]];
            const double gbr = t.gbr, gbc = t.gbc;
            // crossing bin b_f(r, c) = gbr r + gbc c + gg (pos(b_f) == lane)
            double bref;
            float e0f;
            gather_origin(t, r0, c0, &bref, &e0f);
            const double lo = (double)e0f + fmin(0.0, gbr) * (TR - 1) + fmin(0.0, gbc) * (TC - 1);
            const int jlo = (int)floor(lo) - P.cand_half - 1;
            const int bb = (int)bref + jlo;
            // vec: the staged row starts at the 4-aligned bin below bb
            const int shift = P.vec ? bb - (bb & ~3) : 0;
            if (lane == 0) {
                const float stp = t.step_len;
                s_p4[buf][a] = make_float4((float)gbr, (float)gbc, e0f, (float)fabs(t.sigma));
                // shared byte address of local bin 0 minus the floor-trick offset
                const uint32_t ya = stage_u32 +
                                    (uint32_t)((buf * NA + a) * P.slot - jlo + shift) * 4u -
                                    (uint32_t)kMagicBits * 4u;
                s_p2[buf][a] = make_float2(stp, __uint_as_float(ya));
                s_off[buf][a] = shift - jlo;
                s_bb[buf][a] = bb;
            }
        }
    };
    auto prepare_stage = [&](int kb, int buf) {
        const int nc = min(NA, P.n_sel - kb);
        __syncwarp();  // this warp's lane 0 published s_bb
        for (int a = warp; a < nc; a += NW) {
            const int k = kb + a;
            const int bb = s_bb[buf][a];
            const float* yrow = P.y + ((size_t)k * P.Z + z) * P.B;
            const uint32_t dst = stage_u32 + (uint32_t)((buf * NA + a) * P.slot) * 4u;
            if (P.vec) {
                const int bb0 = bb & ~3;
                for (int c = lane; c < (P.slot >> 2); c += 32) {
                    const int bj = bb0 + 4 * c;  // chunks lie fully inside or outside [0, B)
                    const bool ok = bj >= 0 && bj < P.B;
                    cp_async16(dst + (uint32_t)c * 16u, yrow + (ok ? bj : 0), ok ? 16 : 0);
                }
            } else {
                for (int j = lane; j < P.slot; j += 32) {
                    const int bj = bb + j;
                    const bool ok = bj >= 0 && bj < P.B;
                    cp_async4(dst + (uint32_t)j * 4u, yrow + (ok ? bj : 0), ok);
                }
            }
        }
        cp_async_commit();
    };
    auto prepare = [&](int kb, int buf) {
        prepare_params(kb, buf);
        prepare_stage(kb, buf);
    };

    float acc_o[PIX];
#pragma unroll
    for (int j = 0; j < PIX; ++j) acc_o[j] = 0.f;
    f2 rr[PIX / 2];
#pragma unroll
    for (int jj = 0; jj < PIX / 2; ++jj)
        rr[jj] = pk((float)(rg + (2 * jj) * ROWSTEP), (float)(rg + (2 * jj + 1) * ROWSTEP));
    const float clf = (float)cl;
    const f2 mg2 = pk(kMagic, kMagic);

    const int n_chunks = (P.n_sel + NA - 1) / NA;
    if (n_chunks > 0) prepare_params(0, 0);
    pdl_wait<PDL_GATHER>();  // the residual rows are the predecessor's output
    if (n_chunks > 0) prepare_stage(0, 0);
    for (int ci = 0; ci < n_chunks; ++ci) {
        const int buf = (P.nbuf == 2) ? (ci & 1) : 0;
        const int kb = ci * NA;
        const int nc = min(NA, P.n_sel - kb);
        if (P.nbuf == 2 && ci + 1 < n_chunks) {
            prepare(kb + NA, buf ^ 1);
            cp_async_wait_one();
        } else {
            cp_async_wait_all();
        }
        // scale the staged bins by step_len: every lane rescales exactly the
        // elements its own cp.async wrote (complete after its wait), so the
        // CTA barrier below publishes the scaled values
        __syncwarp();
        for (int a = warp; a < nc; a += NW) {
            const float stp = s_p2[buf][a].x;
            float* row = smem + (size_t)(buf * NA + a) * P.slot;
            if (P.vec) {
                float4* row4 = reinterpret_cast<float4*>(row);
                for (int c = lane; c < (P.slot >> 2); c += 32) {
                    float4 q = row4[c];
                    q.x *= stp; q.y *= stp; q.z *= stp; q.w *= stp;
                    row4[c] = q;
                }
            } else {
                for (int j = lane; j < P.slot; j += 32) row[j] *= stp;
            }
        }
        __syncthreads();
        if (TWO_TAP) {
            f2 acc2[PIX / 2];
#pragma unroll
            for (int jj = 0; jj < PIX / 2; ++jj) acc2[jj] = pk(0.f, 0.f);
            auto angle = [&](int a) {
                const float4 q4 = s_p4[buf][a];
                const float2 q2 = s_p2[buf][a];
                const float br = q4.x, S1 = q4.w;
                const float cterm = fmaf(clf, q4.y, q4.z);
                const uint32_t yb = __float_as_uint(q2.y);
                const f2 ct2 = pk(cterm, cterm), br2 = pk(br, br);
                const float nS1 = -S1, oS1 = 1.f - S1;
#pragma unroll
                for (int jj = 0; jj < PIX / 2; ++jj) {
                    const f2 bl = fma2(rr[jj], br2, ct2);
                    const f2 t = add2_rm(bl, mg2);
                    const f2 phi = sub2(bl, sub2(t, mg2));
                    // hat(pos_b - lane) for b = floor(b_f), floor(b_f) + 1 (the
                    // bins carry step_len); saturating FMAs clamp at 0 (<= 1 anyway)
                    float pa, pb, ta, tb, y0a, y1a, y0b, y1b;
                    upk(phi, pa, pb);
                    const f2 w0 = pk(__saturatef(fmaf(nS1, pa, 1.f)),
                                     __saturatef(fmaf(nS1, pb, 1.f)));
                    const f2 w1 = pk(__saturatef(fmaf(S1, pa, oS1)),
                                     __saturatef(fmaf(S1, pb, oS1)));
                    upk(t, ta, tb);
                    lds_pair(mad4(__float_as_uint(ta), yb), y0a, y1a);
                    lds_pair(mad4(__float_as_uint(tb), yb), y0b, y1b);
                    acc2[jj] = fma2(w0, pk(y0a, y0b), fma2(w1, pk(y1a, y1b), acc2[jj]));
                }
            };
            // 8 angles per trip (their shared-memory latencies overlap), then
            // pairs: a subset chunk (30 angles at config 2) has no 1-angle tail loop
            int a = 0;
            for (; a + 8 <= nc; a += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) angle(a + u);
            }
            for (; a + 2 <= nc; a += 2) {
                angle(a);
                angle(a + 1);
            }
            if (a < nc) angle(a);
#pragma unroll
            for (int jj = 0; jj < PIX / 2; ++jj) {
                float a0, a1;
                upk(acc2[jj], a0, a1);
                acc_o[2 * jj] += a0;
                acc_o[2 * jj + 1] += a1;
            }
        } else {
            const float* sl = smem + buf * NA * P.slot;
            float acc_i[PIX];
#pragma unroll
            for (int j = 0; j < PIX; ++j) acc_i[j] = 0.f;
            for (int a = 0; a < nc; ++a) {
                const float4 q4 = s_p4[buf][a];
                const float2 q2 = s_p2[buf][a];
                const float br = q4.x, S1 = q4.w;
                const float cterm = fmaf(clf, q4.y, q4.z);
                const int ybase = a * P.slot + s_off[buf][a] - kMagicBits;
#pragma unroll
                for (int j = 0; j < PIX; ++j) {
                    const float bl = fmaf((float)(rg + j * ROWSTEP), br, cterm);
                    const float tt = __fadd_rd(bl, kMagic);
                    const float phi = bl - (tt - kMagic);
                    const float* yp = sl + (ybase + __float_as_int(tt));
                    for (int q = -P.cand_half + 1; q <= P.cand_half; ++q) {
                        const float w = fmaxf(0.f, 1.f - S1 * fabsf((float)q - phi));
                        acc_i[j] = fmaf(w, yp[q], acc_i[j]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < PIX; ++j) acc_o[j] += acc_i[j];
        }
        if (ci + 1 < n_chunks) __syncthreads();  // buffers are restaged next
    }
    if (n_chunks == 0 && NEPI) {
        cp_async_wait_all();
        __syncthreads();
    }

    const int c = c0 + cl;
    if (c >= P.W) {
        pdl_trigger<PDL_GATHER>();
        return;
    }
    const float* epi = smem + P.nbuf * NA * P.slot;
    const size_t p0 = (size_t)z * plane + (size_t)(r0 + rg) * P.W + c;
#pragma unroll
    for (int j = 0; j < PIX; ++j) {
        const int rl = rg + j * ROWSTEP;
        if (r0 + rl >= P.H) continue;
        const size_t p = p0 + (uint32_t)(j * ROWSTEP * P.W);
        if (EPI == 0) {
            float v = P.alpha * acc_o[j];
            if (P.accumulate) v += P.out[p];
            P.out[p] = v;
        } else {
            const int e = rl * TC + cl;
            step_epilogue_k<EPI>(P.ep, p, acc_o[j], epi[e], epi[TR * TC + e],
                                 NEPI > 2 ? epi[2 * TR * TC + e] : 0.f,
                                 NEPI > 3 ? epi[3 * TR * TC + e] : 0.f);
        }
    }
    pdl_trigger<PDL_GATHER>();
}

__global__ void epilogue_kernel(const float* g, size_t n, pt_step_epilogue ep)
{
    pdl_wait();
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (size_t)gridDim.x * blockDim.x)
        step_epilogue(ep, p, g ? g[p] : 0.f);  // g == null: a zero gradient difference
    pdl_trigger();
}

static constexpr int kNT = 256, kNA = kGatherNA;

template <int TR, int TC, bool TWO, int EPI>
static int run_gather_e(pt_plan* plan, const AdjArgs& a, cudaStream_t st)
{
    const size_t smem = (size_t)(a.nbuf * kNA * a.slot + epi_planes(EPI) * TR * TC) * sizeof(float);
    {
        const int rc = ensure_smem((const void*)adj_gather_kernel<TR, TC, kNT, kNA, TWO, EPI>, smem);
        if (rc) return rc;
    }
    dim3 grid((plan->W + TC - 1) / TC, (plan->H + TR - 1) / TR, plan->Z * a.n_parts);
    PT_CHECK_CUDA(launch_pdl(adj_gather_kernel<TR, TC, kNT, kNA, TWO, EPI>, grid, dim3(kNT), smem,
                             st, a));
    PT_CHECK_LAUNCH();
    return PT_OK;
}

template <int TR, int TC, bool TWO>
static int run_gather_t(pt_plan* plan, const AdjArgs& a, cudaStream_t st)
{
    switch (a.mode == 0 ? 0 : a.n_epi == 2 ? 1 : a.n_epi == 4 ? 2 : 3) {
        case 0: return run_gather_e<TR, TC, TWO, 0>(plan, a, st);
        case 1: return run_gather_e<TR, TC, TWO, 1>(plan, a, st);
        case 2: return run_gather_e<TR, TC, TWO, 2>(plan, a, st);
        default: return run_gather_e<TR, TC, TWO, 3>(plan, a, st);
    }
}

template <bool TWO>
static int run_gather(pt_plan* plan, const AdjArgs& a, cudaStream_t st)
{
    static_assert(kGatherTiles[0][0] == 32 && kGatherTiles[0][1] == 128 &&
                  kGatherTiles[1][0] == 32 && kGatherTiles[1][1] == 64 &&
                  kGatherTiles[2][0] == 16 && kGatherTiles[2][1] == 64 &&
                  kGatherTiles[3][0] == 8 && kGatherTiles[3][1] == 64, "gather tiles");
    switch (plan->gather_tile) {
        case 0: return run_gather_t<32, 128, TWO>(plan, a, st);
        case 1: return run_gather_t<32, 64, TWO>(plan, a, st);
        case 3: return run_gather_t<8, 64, TWO>(plan, a, st);
        default: return run_gather_t<16, 64, TWO>(plan, a, st);
    }
}

// out = alpha * (part_0 + part_1 + ...) (+ out): the angle parts of a split
// adjoint, summed in part order (deterministic)
__global__ void combine_parts_kernel(const float* parts, int n_parts, size_t n, float* out,
                                     float alpha, int accumulate)
{
    pdl_wait();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        float s = parts[i];
        for (int p = 1; p < n_parts; ++p) s += parts[(size_t)p * n + i];
        float v = alpha * s;
        if (accumulate) v += out[i];
        out[i] = v;
    }
    pdl_trigger();
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
    a.vec = (plan->B % 4 == 0) && (((uintptr_t)y & 15) == 0);
    a.slot = a.vec ? ((plan->gather_slot + 3 + 3) & ~3) : plan->gather_slot;
    a.cand_half = plan->cand_half;
    a.nbuf = sel->n > kNA ? 2 : 1;
    a.alpha = alpha;
    a.accumulate = accumulate;
    a.out = x_out;
    a.mode = ep ? 1 : 0;
    if (ep) {
        a.ep = *ep;
        a.n_epi = ep->estimator == PT_EST_SAGA ? 4
                : (ep->estimator == PT_EST_SVRG || ep->estimator == PT_EST_LSVRG) ? 3 : 2;
    } else {
        memset(&a.ep, 0, sizeof(a.ep));
        a.n_epi = 0;
    }
    // A long plain adjoint on an image too small to fill the GPU (config 0's
    // snapshot: 32 tiles x 180 angles) splits its angle chunks over CTAs; the
    // parts land in the workspace's band-partial buffer (free between a
    // forward's reduction and the next forward) and are summed in part order.
    a.n_parts = 1;
    a.chunks_per_part = 0;
    const int n_chunks = (sel->n + kNA - 1) / kNA;
    const int tr = kGatherTiles[plan->gather_tile][0], tc = kGatherTiles[plan->gather_tile][1];
    const long long tiles = (long long)((plan->W + tc - 1) / tc) * ((plan->H + tr - 1) / tr) * plan->Z;
    const size_t npx = (size_t)plan->Z * plan->H * plan->W;
    static const bool split_env = [] {
        const char* e = getenv("PT_GATHER_SPLIT");
        return !(e && e[0] == '0');
    }();
    if (!ep && split_env && ws && n_chunks >= 2 && tiles < plan->sm_count) {
        int parts = (int)std::min<long long>(n_chunks, (2LL * plan->sm_count + tiles - 1) / tiles);
        while (parts > 1 && (size_t)parts * npx > ws->partial_floats) --parts;
        if (parts > 1) {
            a.chunks_per_part = (n_chunks + parts - 1) / parts;
            a.n_parts = (n_chunks + a.chunks_per_part - 1) / a.chunks_per_part;
            a.nbuf = a.chunks_per_part > 1 ? 2 : 1;
            a.out = ws->partial;
            a.alpha = 1.f;
            a.accumulate = 0;
        }
    }
    const int rc = (plan->cand_half == 1) ? run_gather<true>(plan, a, st)
                                          : run_gather<false>(plan, a, st);
    if (rc || a.n_parts == 1) return rc;
    const int blocks = (int)std::min<size_t>((npx + 255) / 256, (size_t)plan->sm_count * 8);
    PT_CHECK_CUDA(launch_pdl(combine_parts_kernel, dim3(blocks), dim3(256), 0, st,
                             (const float*)ws->partial, a.n_parts, npx, x_out, alpha, accumulate));
    PT_CHECK_LAUNCH();
    return PT_OK;
}

int launch_epilogue(pt_plan* plan, const float* g, const pt_step_epilogue* ep, cudaStream_t st)
{
    const size_t n = (size_t)plan->Z * plan->H * plan->W;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)plan->sm_count * 8);
    PT_CHECK_CUDA(launch_pdl(epilogue_kernel, dim3(blocks), dim3(256), 0, st, g, n, *ep));
    PT_CHECK_LAUNCH();
    return PT_OK;
}

}  // namespace pt
