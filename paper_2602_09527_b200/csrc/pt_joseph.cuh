// Device pieces of the projector kernels (projector.cu): the Joseph sample
// loop, the small-image forward's per-segment sums, the gather's tile-origin
// parameters and the fused estimator / ProxSkip epilogue.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "pt_internal.cuh"
#include "pt_simd.cuh"

namespace pt {

// floor() on the fma pipe: x + 1.5*2^23 rounded toward -inf leaves floor(x)
// in the low mantissa bits (valid for |x| < 2^22).
static constexpr float kMagic = 12582912.0f;
static constexpr int kMagicBits = 0x4B400000;

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ float lds(uint32_t a)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
// (x[a], x[a+1]) of a shared-memory address: one IMAD-formed address, two
// loads with an immediate offset
__device__ __forceinline__ void lds_pair(uint32_t a, float& v0, float& v1)
{
    asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+4];"
                 : "=f"(v0), "=f"(v1)
                 : "r"(a));
}
// a*4 + base as one IMAD; `base` is made opaque so the compiler cannot
// re-associate the folded constants back out of it
__device__ __forceinline__ uint32_t mad4(uint32_t a, uint32_t base)
{
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(r) : "r"(a), "r"(base));
    return r;
}
__device__ __forceinline__ uint32_t opaque(uint32_t v)
{
    asm volatile("" : "+r"(v));
    return v;
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const float* src, int valid_bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(valid_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_one() { asm volatile("cp.async.wait_group 1;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;"); }


// Sum of the Joseph samples st in [st_a, st_b) of one ray inside the tile.
// LS / SS: byte strides of one lane / one step in the staged tile.
template <int LS, int SS>
__device__ __forceinline__ float ray_band_sum(uint32_t tile_u32, int st_a, int st_b, float pl,
                                              float mf)
{
    // shared byte address of lane 0 at step st_a, minus the floor-trick
    // magic offset folded in (mod 2^32)
    uint32_t sbase = tile_u32 + (uint32_t)(st_a * SS) - (uint32_t)kMagicBits * (uint32_t)LS;
    const f2 pl2 = pk(pl, pl), m2 = pk(mf, mf), mg2 = pk(kMagic, kMagic);
    const f2 eight2 = pk(8.f, 8.f);
    // a trip = 8 samples as 4 packed pairs (s + u, s + u + 4), u = 0..3: the
    // pair's positions are u*m + (pos(s), pos(s + 4)), so one FFMA2 per pair
    // with a broadcast immediate and no per-pair step counter
    f2 st2 = pk((float)st_a, (float)st_a + 4.f);
    f2 acc2 = pk(0.f, 0.f);
    const int n = st_b - st_a;
    int i = 0;
    for (; i + 8 <= n; i += 8) {
        const uint32_t sb = opaque(sbase);
        const f2 base2 = fma2(st2, m2, pl2);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const f2 pos = u == 0 ? base2 : fma2(pk((float)u, (float)u), m2, base2);
            const f2 t = add2_rm(pos, mg2);
            const f2 fr = sub2(pos, sub2(t, mg2));
            float ta, tb, a0, a1, b0, b1;
            upk(t, ta, tb);
            const uint32_t aa = __float_as_uint(ta) * (uint32_t)LS + sb + u * SS;
            const uint32_t ab = __float_as_uint(tb) * (uint32_t)LS + sb + (u + 4) * SS;
            asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+%3];"
                         : "=f"(a0), "=f"(a1) : "r"(aa), "n"(LS));
            asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+%3];"
                         : "=f"(b0), "=f"(b1) : "r"(ab), "n"(LS));
            const f2 x0 = pk(a0, b0), x1 = pk(a1, b1);
            acc2 = add2(acc2, fma2(fr, sub2(x1, x0), x0));
        }
        st2 = add2(st2, eight2);
        sbase += 8 * SS;
    }
    float acc0, acc1;
    upk(acc2, acc0, acc1);
    float sa, sb_;
    upk(st2, sa, sb_);
    for (; i < n; ++i) {
        const float pa = fmaf(sa, mf, pl);
        const float ta = __fadd_rd(pa, kMagic);
        const float fa = pa - (ta - kMagic);
        const uint32_t aa = __float_as_uint(ta) * (uint32_t)LS + opaque(sbase);
        float a0, a1;
        asm volatile("ld.shared.f32 %0, [%2];\n\tld.shared.f32 %1, [%2+%3];"
                     : "=f"(a0), "=f"(a1) : "r"(aa), "n"(LS));
        acc0 += fmaf(fa, a1 - a0, a0);
        sa += 1.f;
        sbase += SS;
    }
    return acc0 + acc1;
}

// ---------------------------------------------------------------------------
// Small images (both sides <= 128, Z = 1; config 0 is 128^2): the whole image
// is staged in a zero-margined buffer [132][133] (image (0, 0) at (2, 2): both
// taps of every clipped sample lie inside it; the odd pitch puts a
// column-stepping warp's lanes in distinct banks).  A ray is summed in
// kSmallNseg segments of kSmallSeg steps (float32 inside a segment), the
// segments combined in float64 in segment order (the band partials' scheme,
// SURVEY.md 7.3.1).
// ---------------------------------------------------------------------------
constexpr int kSmallMax = 128, kSmallMargin = 2;
constexpr int kSmallRows = kSmallMax + 2 * kSmallMargin;       // 132
constexpr int kSmallPitch = (kSmallMax + 2 * kSmallMargin) | 1;  // 133 (cp.async staging)
// one TMA box: x origin -4 (a box's innermost coordinate must be 16-byte
// aligned), so 4 zero columns on the left; 136 columns cover -4 .. 131
constexpr int kSmallPitchT = kSmallMax + 8;                      // 136
constexpr int kSmallSmem = kSmallRows * kSmallPitchT * 4;       // either layout fits
// columns left of image column 0 in a layout of this pitch
template <int PITCH>
constexpr int small_mx() { return PITCH == kSmallPitchT ? 4 : kSmallMargin; }
constexpr int kSmallSeg = 8, kSmallNseg = kSmallMax / kSmallSeg;

// Threads [t0, t0 + nthr) (whole warps) copy the image into the staged buffer.
__device__ __forceinline__ void small_stage(const float* x, int H, int W, uint32_t buf, int t0,
                                            int nthr)
{
    const int lane = threadIdx.x & 31, w0 = (threadIdx.x - t0) >> 5, nw = nthr >> 5;
    for (int r = w0; r < kSmallRows; r += nw) {
        const int gi = r - kSmallMargin;
        const bool rin = gi >= 0 && gi < H;
        const float* src = x + (size_t)(rin ? gi : 0) * W;
        for (int c = lane; c < kSmallPitch; c += 32) {
            const int gj = c - kSmallMargin;
            const bool ok = rin && gj >= 0 && gj < W;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                             buf + (uint32_t)(r * kSmallPitch + c) * 4u),
                         "l"(src + (ok ? gj : 0)), "r"(ok ? 4 : 0));
        }
    }
}

// The whole image by one TMA box (136 x 132 from (-4, -2): the copy engine
// zero-fills outside the image) into the dense [132][136] layout, completion
// on `bar` (initialised by the caller); one thread issues.  W % 4 == 0.
__device__ __forceinline__ void small_stage_tma(const CUtensorMap* map, uint32_t buf, uint32_t bar)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                 "r"((uint32_t)(kSmallRows * kSmallPitchT * 4)) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(buf),
        "l"(map), "r"(-4), "r"(-kSmallMargin), "r"(bar) : "memory");
}
__device__ __forceinline__ void small_mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SW_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}

// One ray of one angle: lane position at step 0 (float64 -> float32), slope.
struct SmallRay {
    float pl, mf, im;
    int branch, n_steps, n_lanes;
};
__device__ __forceinline__ SmallRay small_ray(const AngleTab& t, int b, int H, int W)
{
    SmallRay r;
    r.pl = (float)__fma_rn((double)b, t.sigma, t.a0);
    r.mf = (float)t.m;
    r.im = (float)t.im;
    r.branch = t.branch;
    r.n_steps = t.branch ? W : H;
    r.n_lanes = t.branch ? H : W;
    return r;
}
// Float32 sum of segment `seg` of the ray over the staged buffer: the steps
// of the segment where pos in [-1.5, n_lanes + 0.5] (outside, both taps are
// zero, as in fwd_band_kernel).
template <int PITCH>
__device__ __forceinline__ float small_segment(uint32_t buf, const SmallRay& r, int seg)
{
    int st_a = seg * kSmallSeg, st_b = min(r.n_steps, st_a + kSmallSeg);
    if (r.im == 0.f) {
        if (r.pl < -1.5f || r.pl > r.n_lanes + 0.5f) st_b = 0;
    } else {
        const float e1 = __fmul_rn(-1.5f - r.pl, r.im);
        const float e2 = __fmul_rn((float)r.n_lanes + 0.5f - r.pl, r.im);
        const float lo = fminf(e1, e2), hi = fmaxf(e1, e2);
        st_a = max(st_a, (int)ceilf(fminf(fmaxf(lo, -1.f), (float)kSmallMax + 1.f)));
        st_b = min(st_b, (int)floorf(fminf(fmaxf(hi, -2.f), (float)kSmallMax + 1.f)) + 1);
    }
    if (st_a >= st_b) return 0.f;
    // image (0, 0) at buffer row kSmallMargin, column small_mx<PITCH>()
    const uint32_t org = buf + (uint32_t)(kSmallMargin * PITCH + small_mx<PITCH>()) * 4u;
    return r.branch == 0 ? ray_band_sum<4, PITCH * 4>(org, st_a, st_b, r.pl, r.mf)
                         : ray_band_sum<PITCH * 4, 4>(org, st_a, st_b, r.pl, r.mf);
}
// Line integral of a ray from its segments' sums (float64, in segment
// order), and its residual row value (operations pinned: no contraction)
__device__ __forceinline__ double small_line_integral(const float* seg_sums, int stride,
                                                      float step_len)
{
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < kSmallNseg; ++g) s = __dadd_rn(s, (double)seg_sums[g * stride]);
    return __dmul_rn(s, (double)step_len);
}
__device__ __forceinline__ float residual_value(double yd, const float* data, const float* data2,
                                                size_t o)
{
    if (data) yd = __dsub_rn(yd, (double)data[o]);
    if (data2) yd = __dsub_rn(yd, (double)data2[o]);
    return (float)yd;
}

// Gather: the crossing bin of the tile origin (r0, c0), b_f = gbr r0 + gbc c0
// + gg, as its floor and the float32 fraction (the tile frame of every
// pixel's two-tap lookup).
__device__ __forceinline__ void gather_origin(const AngleTab& t, int r0, int c0, double* bref,
                                              float* e0)
{
    const double bf00 = __fma_rn(t.gbr, (double)r0, __fma_rn(t.gbc, (double)c0, t.gg));
    *bref = floor(bf00);
    *e0 = (float)(bf00 - *bref);
}

// Gather epilogue kinds (compile-time): 0 plain adjoint, 1 full/sgd, 2 saga,
// 3 svrg/lsvrg; the number of operand planes prefetched for each
__host__ __device__ constexpr int epi_planes(int epi)
{
    return epi == 0 ? 0 : epi == 1 ? 2 : epi == 2 ? 4 : 3;
}

// step_epilogue_vals with the estimator class fixed at compile time (the
// per-pixel epilogue of the gather; same expressions, same operation order)
template <int EPI>
__device__ __forceinline__ void step_epilogue_k(const pt_step_epilogue& ep, size_t p, float g,
                                                float xv, float hv, float a0v, float a1v)
{
    float est;
    if (EPI == 1) {
        est = ep.estimator == PT_EST_FULL ? g : ep.n_scale * g;
    } else if (EPI == 2) {
        est = ep.n_scale * g + (a1v - ep.n_scale * a0v);
        ep.aux1[p] = (a1v - a0v) + g;
        ep.aux0[p] = g;
    } else {
        est = ep.n_scale * g + a0v;
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


}  // namespace pt
