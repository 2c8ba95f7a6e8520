// FGP (Beck-Teboulle fast gradient projection on the dual) TV prox for
// sm_100a, temporally blocked: one launch runs T inner iterations on a
// (RH x RW) region held on chip, of which the central (RH-2T) x (RW-2T)
// points are exact after T iterations (each iteration's stencil reaches one
// point further, pkg/src/proxtomo/regularizers.py:62-76; the final launch's
// x = v - lam D^T(p, q) needs one ring more); only those are written back.  So a prox call with n inner iterations costs ceil(n/T)
// HBM round trips of the dual state instead of n.
//
// Per-iteration math (regularizers.py:112-129), lam = tau*alpha, eta = 1/(8 lam):
//   u  = v - lam D^T(r, s);  u = max(u, 0) if nonneg
//   (ph, qh) = (r, s) + eta D u
//   (p', q') = (ph, qh) / max(1, |(ph, qh)|)
//   (r, s)   = (p', q') + beta_k ((p', q') - (p, q));  (p, q) = (p', q')
// and the output (:130-132) x = max(v - lam D^T(p, q), 0).
//
// Layout: each thread owns a vertical strip of STRIP points of one column;
// v, p, q, r, s, u of its points live in registers.  Only the values a
// neighbour needs cross threads: s and u through shared-memory planes
// (left / right neighbours), r and u of the strip ends through two small
// row buffers (up / down neighbours).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "pt_internal.cuh"
#include "pt_simd.cuh"

namespace pt {

constexpr int kFgpMaxT = 12;  // inner iterations per launch (2D)

struct FgpArgs {
    int H, W;  // the image (H = global rows)
    // the arrays hold rows [grow0, grow0 + Ha) of the image (row slab with
    // ghost rows; the whole image: grow0 = 0, Ha = H); outputs are the array
    // rows [row_lo, row_lo + rows_out) (final outputs indexed from row_lo)
    int Ha, grow0, row_lo, rows_out;
    const float* v;
    const float *p_in, *q_in, *r_in, *s_in;  // r_in == nullptr: r = p, s = q (call start)
    float *p_out, *q_out, *r_out, *s_out;
    float lam, eta;
    float beta[kFgpMaxT];
    int n_iter;
    int halo;
    int nonneg;
    int final_;
    float* x_out;
    const float* xhat;
    float* h;
    float pog;
    long long iteration;
    long long* bad_iter;
};

__device__ __forceinline__ float rsqrt_ftz(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// max that propagates NaN (max.NaN): the divergence check must see NaN duals
__device__ __forceinline__ float max_nan(float a, float b)
{
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
// Interior iteration with packed f32x2 arithmetic.  A thread's strip rows are
// held as pairs (j, j + H2), H2 = STRIP/2, so the up-neighbour of pair j is
// pair j-1 and the down-neighbour of pair j is pair j+1 (one repack at the
// strip ends): the stencil needs no lane shuffling.  The left/right exchange
// planes store the pairs as float2 (one 64-bit LDS/STS per pair, operands land
// in aligned register pairs).
__device__ __forceinline__ f2 ld2(const float2* p)
{
    f2 r;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r.v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return r;
}
__device__ __forceinline__ void st2(float2* p, f2 v)
{
    asm volatile("st.shared.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "l"(v.v));
}

// per-half select of two pairs: (clo ? lo(a) : lo(b), chi ? hi(a) : hi(b))
__device__ __forceinline__ f2 sel2(f2 a, f2 b, bool clo, bool chi)
{
    float al, ah, bl, bh;
    upk(a, al, ah);
    upk(b, bl, bh);
    return pk(clo ? al : bl, chi ? ah : bh);
}

// EDGE = the region touches the image border (or the arrays' row range): the
// same packed arithmetic, with the boundary rules of fgp2d_iteration applied
// by per-half selects -- lr_mask bit k: strip row k is above the image's last
// row (D's vertical difference and D^T's -r term exist), in_mask bit k: the
// point is inside the image, nlc: the column is not the image's last.  A point
// inside the image and off its last row / column evaluates exactly the
// interior expressions, so edge and interior regions agree bitwise.
template <int RW, int RH, int STRIP, bool NONNEG, bool EDGE = false>
__device__ __forceinline__ void fgp2d_iteration_packed(
    f2 (&V)[STRIP / 2], f2 (&Pp)[STRIP / 2], f2 (&Q)[STRIP / 2], f2 (&R)[STRIP / 2],
    f2 (&S)[STRIP / 2], f2 (&U)[STRIP / 2], float2 (*S_s2)[RW + 2], float2 (*S_u2)[RW + 2],
    float (*S_r)[RW], float (*S_ut)[RW], int tx, int ty, float lam, float eta, float beta,
    unsigned in_mask = 0u, unsigned lr_mask = 0u, bool nlc = true)
{
    constexpr int H2 = STRIP / 2;
    const int prow0 = ty * H2;
    const f2 nlam2 = pk(-lam, -lam), eta2 = pk(eta, eta), beta2 = pk(beta, beta);
    const f2 z2 = pk(0.f, 0.f);
    auto in_ = [&](int k) { return ((in_mask >> k) & 1u) != 0u; };
    auto lr_ = [&](int k) { return ((lr_mask >> k) & 1u) != 0u; };
#pragma unroll
    for (int j = 0; j < H2; ++j) st2(&S_s2[prow0 + j][tx + 1], S[j]);
    S_r[ty + 1][tx] = hi_of(R[H2 - 1]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < H2; ++j) {
        // zero padding (row 0 of S_r, column 0 of S_s2) stands for the region edge
        const f2 r_up = j ? R[j - 1] : pk(S_r[ty][tx], lo_of(R[H2 - 1]));
        const f2 s_left = ld2(&S_s2[prow0 + j][tx]);
        // _diff_adjoint (regularizers.py:70-76): ((-r + r_up) - s) + s_left
        f2 o = sub2(r_up, R[j]);
        if (EDGE) o = sel2(o, r_up, lr_(j), lr_(j + H2));
        const f2 os = sub2(o, S[j]);
        o = (!EDGE || nlc) ? os : o;
        o = add2(o, s_left);
        f2 u = fma2(nlam2, o, V[j]);
        if (NONNEG) {
            float ua, ub;
            upk(u, ua, ub);
            u = pk(max_nan(ua, 0.f), max_nan(ub, 0.f));  // NaN propagates
        }
        if (EDGE) u = sel2(u, z2, in_(j), in_(j + H2));
        U[j] = u;
        st2(&S_u2[prow0 + j][tx + 1], u);
    }
    S_ut[ty][tx] = lo_of(U[0]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < H2; ++j) {
        // rows (j+1, j+1+H2); for the last pair: (pair 0 hi, next strip's first row)
        const f2 u_down = (j < H2 - 1) ? U[j + 1] : pk(hi_of(U[0]), S_ut[ty + 1][tx]);
        const f2 u_right = ld2(&S_u2[prow0 + j][tx + 2]);
        f2 gv = sub2(u_down, U[j]);
        f2 gh = sub2(u_right, U[j]);
        if (EDGE) {
            gv = sel2(gv, z2, lr_(j), lr_(j + H2));
            gh = nlc ? gh : z2;
        }
        const f2 ph = fma2(eta2, gv, R[j]);
        const f2 qh = fma2(eta2, gh, S[j]);
        const f2 n2 = fma2(ph, ph, mul2(qh, qh));
        float na, nb;
        upk(n2, na, nb);
        // 1 / max(1, |.|): rsqrt of max(n2, 1) (exactly 1 at 1; NaN propagates)
        const f2 inv = pk(rsqrt_ftz(max_nan(na, 1.f)), rsqrt_ftz(max_nan(nb, 1.f)));
        const f2 pn = mul2(ph, inv), qn = mul2(qh, inv);
        const f2 rn = fma2(beta2, sub2(pn, Pp[j]), pn);
        const f2 sn = fma2(beta2, sub2(qn, Q[j]), qn);
        if (EDGE) {
            const bool a = in_(j), b = in_(j + H2);
            R[j] = sel2(rn, R[j], a, b);
            S[j] = sel2(sn, S[j], a, b);
            Pp[j] = sel2(pn, Pp[j], a, b);
            Q[j] = sel2(qn, Q[j], a, b);
        } else {
            R[j] = rn;
            S[j] = sn;
            Pp[j] = pn;
            Q[j] = qn;
        }
    }
}

template <int RW, int RH, int STRIP, bool NONNEG>
__global__ void __launch_bounds__(RW*(RH / STRIP), 2) fgp2d_kernel(FgpArgs P)
{
    constexpr int H2 = STRIP / 2, NS = RH / STRIP, PW = RW + 2;
    // exchange planes, pitch RW + 2: a thread's column at tx + 1, columns 0 and
    // RW + 1 hold zeros (the region edge).  The scalar (edge / epilogue) and the
    // pair (interior) layouts share one buffer; a CTA uses one at a time and
    // re-zeroes the padding when it switches.
    __shared__ __align__(16) float S_buf[2 * RH * PW];
    float (*S_s)[PW] = reinterpret_cast<float (*)[PW]>(S_buf);
    float (*S_u)[PW] = reinterpret_cast<float (*)[PW]>(S_buf + RH * PW);
    float2 (*S_s2)[PW] = reinterpret_cast<float2 (*)[PW]>(S_buf);
    float2 (*S_u2)[PW] = reinterpret_cast<float2 (*)[PW]>(S_buf + RH * PW);
    // strip-end rows: S_r row ty + 1 = last r of strip ty (row 0 zero),
    // S_ut row ty = first u of strip ty (row NS zero)
    __shared__ float S_r[NS + 1][RW];
    __shared__ float S_ut[NS + 1][RW];

    const int tid = threadIdx.x;
    const int tx = tid % RW;
    const int ty = tid / RW;
    const int IW = RW - 2 * P.halo, IH = RH - 2 * P.halo;
    const int j0 = blockIdx.x * IW - P.halo;
    const int i0 = P.row_lo + blockIdx.y * IH - P.halo;  // array row of the region
    const int gi0 = i0 + P.grow0;                          // its image row
    const int gj = j0 + tx;
    const int row0 = ty * STRIP;
    const bool col_in = (gj >= 0 && gj < P.W);
    const bool not_last_col = (gj < P.W - 1);
    // the whole region, and one point beyond it, strictly inside the image
    // (and inside the arrays)
    const bool edge = !(gi0 >= 0 && j0 >= 0 && gi0 + RH < P.H && j0 + RW < P.W && i0 >= 0 &&
                        i0 + RH <= P.Ha);

    auto zero_pads = [&](bool packed) {
        // rows of the active layout: RH scalar rows or RH / 2 pair rows, 2 planes
        const int rows = packed ? RH / 2 : RH;
        for (int i = tid; i < 4 * rows; i += RW * NS) {
            const int plane = i / (2 * rows), rr = (i >> 1) % rows, side = i & 1;
            float* base = S_buf + plane * RH * PW;
            if (packed) {
                float2* row = reinterpret_cast<float2*>(base) + rr * PW;
                row[side ? RW + 1 : 0] = make_float2(0.f, 0.f);
            } else {
                base[rr * PW + (side ? RW + 1 : 0)] = 0.f;
            }
        }
    };
    zero_pads(true);
    if (tid < RW) {
        S_r[0][tid] = 0.f;
        S_ut[NS][tid] = 0.f;
    }

    pdl_wait<PDL_FGP2D>();
    // packed state: pair j = strip rows (j, j + H2)
    f2 V[H2], Pp[H2], Q[H2], R[H2], S[H2], U[H2];
    unsigned in_mask = 0;
    if (!edge) {
        // every point inside the image: unpredicated loads, all in flight
        in_mask = (1u << STRIP) - 1u;
        const size_t base = (size_t)(i0 + row0) * P.W + gj;
        const size_t W = P.W;
        float vv[STRIP], pv[STRIP], qv[STRIP], rv[STRIP], sv[STRIP];
#pragma unroll
        for (int k = 0; k < STRIP; ++k) {
            vv[k] = P.v[base + k * W];
            pv[k] = P.p_in[base + k * W];
            qv[k] = P.q_in[base + k * W];
        }
        if (P.r_in) {
#pragma unroll
            for (int k = 0; k < STRIP; ++k) {
                rv[k] = P.r_in[base + k * W];
                sv[k] = P.s_in[base + k * W];
            }
        } else {
#pragma unroll
            for (int k = 0; k < STRIP; ++k) {
                rv[k] = pv[k];
                sv[k] = qv[k];
            }
        }
#pragma unroll
        for (int j = 0; j < H2; ++j) {
            V[j] = pk(vv[j], vv[j + H2]);
            Pp[j] = pk(pv[j], pv[j + H2]);
            Q[j] = pk(qv[j], qv[j + H2]);
            R[j] = pk(rv[j], rv[j + H2]);
            S[j] = pk(sv[j], sv[j + H2]);
            U[j] = pk(0.f, 0.f);
        }
    } else {
#pragma unroll
        for (int j = 0; j < H2; ++j) {
            float vv[2], pv[2], qv[2], rv[2], sv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int k = j + h * H2;
                const int ai = i0 + row0 + k, gi = ai + P.grow0;
                const bool in = col_in && gi >= 0 && gi < P.H && ai >= 0 && ai < P.Ha;
                if (in) in_mask |= 1u << k;
                const size_t o = in ? (size_t)ai * P.W + gj : 0;
                vv[h] = in ? P.v[o] : 0.f;
                pv[h] = in ? P.p_in[o] : 0.f;
                qv[h] = in ? P.q_in[o] : 0.f;
                rv[h] = in ? (P.r_in ? P.r_in[o] : pv[h]) : 0.f;
                sv[h] = in ? (P.s_in ? P.s_in[o] : qv[h]) : 0.f;
            }
            V[j] = pk(vv[0], vv[1]);
            Pp[j] = pk(pv[0], pv[1]);
            Q[j] = pk(qv[0], qv[1]);
            R[j] = pk(rv[0], rv[1]);
            S[j] = pk(sv[0], sv[1]);
            U[j] = pk(0.f, 0.f);
        }
    }
    if (!edge) {
        // two iterations per trip: the compiler alternates register roles instead of moving
        int it = 0;
        for (; it + 1 < P.n_iter; it += 2) {
            fgp2d_iteration_packed<RW, RH, STRIP, NONNEG>(V, Pp, Q, R, S, U, S_s2, S_u2, S_r, S_ut,
                                                          tx, ty, P.lam, P.eta, P.beta[it]);
            fgp2d_iteration_packed<RW, RH, STRIP, NONNEG>(V, Pp, Q, R, S, U, S_s2, S_u2, S_r, S_ut,
                                                          tx, ty, P.lam, P.eta, P.beta[it + 1]);
        }
        if (it < P.n_iter)
            fgp2d_iteration_packed<RW, RH, STRIP, NONNEG>(V, Pp, Q, R, S, U, S_s2, S_u2, S_r, S_ut,
                                                          tx, ty, P.lam, P.eta, P.beta[it]);
    } else {
        // the same packed iteration with the boundary rules as per-half selects
        // (bit k of lr_mask: image row of strip row k below H - 1)
        const int last_k = P.H - 1 - (gi0 + row0);  // strip rows k < last_k are above the last row
        const unsigned lr_mask =
            last_k <= 0 ? 0u : (last_k >= STRIP ? (1u << STRIP) - 1u : (1u << last_k) - 1u);
        for (int it = 0; it < P.n_iter; ++it)
            fgp2d_iteration_packed<RW, RH, STRIP, NONNEG, true>(
                V, Pp, Q, R, S, U, S_s2, S_u2, S_r, S_ut, tx, ty, P.lam, P.eta, P.beta[it],
                in_mask, lr_mask, not_last_col);
    }

    float v[STRIP], p[STRIP], q[STRIP], r[STRIP], s[STRIP];
#pragma unroll
    for (int j = 0; j < H2; ++j) {
        upk(V[j], v[j], v[j + H2]);
        upk(Pp[j], p[j], p[j + H2]);
        upk(Q[j], q[j], q[j + H2]);
        upk(R[j], r[j], r[j + H2]);
        upk(S[j], s[j], s[j + H2]);
    }
    // exact points: the region minus its halo, inside the image
    const bool col_inner = tx >= P.halo && tx < RW - P.halo && col_in;
    // exact rows of the region that are output rows
    const int k_lo = max(max(0, P.halo - row0), P.row_lo - (i0 + row0));
    const int k_hi = min(min(STRIP, RH - P.halo - row0), P.row_lo + P.rows_out - (i0 + row0));
    const size_t obase = (size_t)(i0 + row0) * P.W + gj;           // array index
    const size_t fbase = obase - (size_t)P.row_lo * P.W;           // final outputs
    const float lam = P.lam;
    if (P.final_) {
        // x = max(v - lam D^T(p, q), 0), then the ProxSkip h update
        __syncthreads();
        zero_pads(false);
#pragma unroll
        for (int k = 0; k < STRIP; ++k) S_s[row0 + k][tx + 1] = q[k];
        S_r[ty + 1][tx] = p[STRIP - 1];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < STRIP; ++k) {
            const int gi = gi0 + row0 + k;
            if (!col_inner || k < k_lo || k >= k_hi || !((in_mask >> k) & 1u)) continue;
            const float p_up = k ? p[k - 1] : S_r[ty][tx];
            const float q_left = S_s[row0 + k][tx];
            float o = (gi < P.H - 1) ? -p[k] : 0.f;
            o += p_up;
            o = not_last_col ? o - q[k] : o;
            o += q_left;
            float x = v[k] - lam * o;
            if (NONNEG) x = (x < 0.f) ? 0.f : x;
            const size_t idx = fbase + (size_t)k * P.W;
            P.x_out[idx] = x;
            P.p_out[idx] = p[k];
            P.q_out[idx] = q[k];
            if (P.h) {
                P.h[idx] = P.h[idx] + P.pog * (x - P.xhat[idx]);
            }
            if (!isfinite(x) && P.bad_iter) atomicMin(P.bad_iter, P.iteration);
        }
    } else {
#pragma unroll
        for (int k = 0; k < STRIP; ++k) {
            if (!col_inner || k < k_lo || k >= k_hi || !((in_mask >> k) & 1u)) continue;
            const size_t idx = obase + (size_t)k * P.W;
            P.p_out[idx] = p[k];
            P.q_out[idx] = q[k];
            P.r_out[idx] = r[k];
            P.s_out[idx] = s[k];
        }
    }
    pdl_trigger<PDL_FGP2D>();
}

int64_t fgp_workspace_floats(const pt_plan* plan)
{
    // two ping-pong sets of (p, q, r, s) [2D] or (p, q, w, r, s, t) [3D]
    if (plan->Z > 1) return fgp3d_slab_floats(plan->Z, plan->H, plan->W);
    return 8 * (int64_t)plan->H * plan->W;
}

// 64 x 64 regions (T up to 8) from 256 x 256 images up, 32 x 32 regions with
// T = 10 below (PT_FGP_BIG_MIN: the smallest min(H, W) that uses 64 x 64
// regions; PT_FGP_T_SMALL: T of the 32 x 32 regions).  A 128^2 image is
// latency bound: 32 x 32 regions with a 10-ring halo give 121 CTAs per launch
// (64 x 64 regions: 9) and five launches per FGP-50: 82 -> 50 us.
static bool fgp2d_big(int H, int W)
{
    static const int big_min = [] {
        const char* e = getenv("PT_FGP_BIG_MIN");
        return e ? atoi(e) : 256;
    }();
    return std::min(H, W) >= big_min;
}

// inner iterations per launch of the 64 x 64 regions (PT_FGP_T overrides).
// The result does not depend on T (exact points only), the time does, through
// launches x ragged last regions x waves; FGP-100 with the T-ring halo:
// 2048^2 T = 8 0.996 ms (T = 5 / 6 / 7 / 9..12: 1.01-1.19 ms), 512^2 T = 8
// 156 us (T = 5 / 6 / 7: 188 / 174 / 166 us).
static int fgp2d_tmax(int H, int W)
{
    static const int env = [] {
        const char* e = getenv("PT_FGP_T");
        return e ? std::max(1, std::min(kFgpMaxT, atoi(e))) : 0;
    }();
    (void)H;
    (void)W;
    return env ? env : 8;
}

template <int RW, int RH, int STRIP>
static int run_fgp2d(pt_plan* plan, const float* v, double lam, int inner, int nonneg, float* p,
                     float* q, float* x_out, const float* xhat, float* h, float pog,
                     int64_t iteration, int64_t* bad_iter, float* work, cudaStream_t st,
                     int tmax)
{
    const size_t n = (size_t)plan->H * plan->W;
    float* X[4] = {work, work + n, work + 2 * n, work + 3 * n};
    float* Y[4] = {work + 4 * n, work + 5 * n, work + 6 * n, work + 7 * n};
    // momentum sequence: t restarts at 1 every call (regularizers.py:109,125-126)
    std::vector<double> betas(inner);
    double t = 1.0;
    for (int k = 0; k < inner; ++k) {
        const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        betas[k] = (t - 1.0) / tn;
        t = tn;
    }
    // at least two exact points per region side on the final launch (halo T + 1)
    tmax = std::max(1, std::min(tmax, (std::min(RW, RH) - 3) / 2));
    const int n_launch = (inner + tmax - 1) / tmax;
    const float *sp = p, *sq = q, *sr = nullptr, *ss = nullptr;
    if (n_launch == 1) {
        PT_CHECK_CUDA(cudaMemcpyAsync(X[0], p, n * 4, cudaMemcpyDeviceToDevice, st));
        PT_CHECK_CUDA(cudaMemcpyAsync(X[1], q, n * 4, cudaMemcpyDeviceToDevice, st));
        sp = X[0];
        sq = X[1];
    }
    int done = 0;
    for (int L = 0; L < n_launch; ++L) {
        const int iters = std::min(tmax, inner - done);
        const bool fin = (L == n_launch - 1);
        FgpArgs a;
        a.H = plan->H;
        a.W = plan->W;
        a.Ha = plan->H; a.grow0 = 0; a.row_lo = 0; a.rows_out = plan->H;
        a.v = v;
        a.p_in = sp; a.q_in = sq; a.r_in = sr; a.s_in = ss;
        float** D = (L % 2 == 0) ? Y : X;
        if (fin) {
            a.p_out = p; a.q_out = q; a.r_out = nullptr; a.s_out = nullptr;
        } else {
            a.p_out = D[0]; a.q_out = D[1]; a.r_out = D[2]; a.s_out = D[3];
        }
        a.lam = (float)lam;
        a.eta = (float)(1.0 / (8.0 * lam));
        for (int k = 0; k < kFgpMaxT; ++k) a.beta[k] = (k < iters) ? (float)betas[done + k] : 0.f;
        a.n_iter = iters;
        // T iterations make T rings of the region inexact (each iteration's
        // stencil reaches one point in every direction); the final launch's
        // x = v - lam D^T(p, q) needs one ring more
        a.halo = fin ? iters + 1 : iters;
        a.nonneg = nonneg;
        a.final_ = fin ? 1 : 0;
        a.x_out = x_out;
        a.xhat = xhat;
        a.h = h;
        a.pog = pog;
        a.iteration = (long long)iteration;
        a.bad_iter = (long long*)bad_iter;
        const int IW = RW - 2 * a.halo, IH = RH - 2 * a.halo;
        dim3 grid((plan->W + IW - 1) / IW, (plan->H + IH - 1) / IH);
        PT_CHECK_CUDA(launch_pdl(nonneg ? fgp2d_kernel<RW, RH, STRIP, true>
                                        : fgp2d_kernel<RW, RH, STRIP, false>,
                                 grid, dim3(RW * (RH / STRIP)), 0, st, a));
        PT_CHECK_LAUNCH();
        if (!fin) {
            sp = D[0]; sq = D[1]; sr = D[2]; ss = D[3];
        }
        done += iters;
    }
    return PT_OK;
}

// ---------------------------------------------------------------------------
// Row slabs of a 2D image (multi-GPU "rows" decomposition):
// slab g owns image rows [r0, r0 + Hl).  Its FGP state lives in extended
// arrays of Ha = Hl + 2 G rows (G = kRowGhost ghost rows above and below);
// before every launch the ghost rows hold the neighbours' boundary rows, so
// the launch's T <= G - 1 iterations on the slab's own rows see exactly the
// values the whole-image launch sees: the result is bitwise the whole-image
// result (edge and interior regions evaluate identical expressions).
// Workspace per slab: v, (p, q, r, s) x 2, each Ha x W.
// ---------------------------------------------------------------------------
int64_t fgp2d_slab_floats(int Hl, int W) { return 9 * (int64_t)(Hl + 2 * kRowGhost) * W; }

namespace {
struct RowSets {
    float* a[9];  // v, X[0..3], Y[0..3]
};
RowSets row_sets(const Fgp2Slab& s, int W)
{
    RowSets r;
    const size_t n = (size_t)(s.Hl + 2 * kRowGhost) * W;
    for (int i = 0; i < 9; ++i) r.a[i] = s.work + i * n;
    return r;
}
}  // namespace

// ghost rows of arrays `first .. first + n - 1` of every slab's sets
static int fgp2d_rows_exchange(const Fgp2Slab* sl, int G, int W, int first, int n,
                               const RowHalo* halo, cudaStream_t st)
{
    const int GR = kRowGhost;
    const size_t band = (size_t)GR * W * 4;
    for (int g = 0; g + 1 < G; ++g) {
        const RowSets lo = row_sets(sl[g], W), hi = row_sets(sl[g + 1], W);
        const int Hl = sl[g].Hl;
        for (int i = first; i < first + n; ++i) {
            // lower slab's bottom ghost rows <- upper slab's first own rows
            PT_CHECK_CUDA(cudaMemcpyAsync(lo.a[i] + (size_t)(GR + Hl) * W, hi.a[i] + (size_t)GR * W,
                                          band, cudaMemcpyDeviceToDevice, st));
            // upper slab's top ghost rows <- lower slab's last own rows
            PT_CHECK_CUDA(cudaMemcpyAsync(hi.a[i], lo.a[i] + (size_t)Hl * W, band,
                                          cudaMemcpyDeviceToDevice, st));
        }
    }
    if (halo && halo->world > 1) {
        const RowSets r = row_sets(sl[0], W);
        return halo->exchange(halo->ctx, n, r.a + first, sl[0].Hl, W, GR, st);
    }
    return PT_OK;
}

template <int RW, int RH, int STRIP>
static int fgp2d_rows_run_t(const Fgp2Slab* sl, int G, int H, int W, double lam, int inner,
                            int nonneg, float pog, int64_t iteration, int64_t* bad_iter,
                            const RowHalo* halo, int tmax, cudaStream_t st)
{
    const int GR = kRowGhost;
    std::vector<double> betas(inner);
    double t = 1.0;
    for (int k = 0; k < inner; ++k) {
        const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        betas[k] = (t - 1.0) / tn;
        t = tn;
    }
    // own rows of v, p, q into the extended arrays, then their ghost rows
    for (int g = 0; g < G; ++g) {
        const RowSets r = row_sets(sl[g], W);
        const size_t off = (size_t)GR * W, n = (size_t)sl[g].Hl * W * 4;
        PT_CHECK_CUDA(cudaMemcpyAsync(r.a[0] + off, sl[g].v, n, cudaMemcpyDeviceToDevice, st));
        PT_CHECK_CUDA(cudaMemcpyAsync(r.a[1] + off, sl[g].p, n, cudaMemcpyDeviceToDevice, st));
        PT_CHECK_CUDA(cudaMemcpyAsync(r.a[2] + off, sl[g].q, n, cudaMemcpyDeviceToDevice, st));
    }
    int rc = fgp2d_rows_exchange(sl, G, W, 0, 3, halo, st);
    if (rc) return rc;
    const int n_launch = (inner + tmax - 1) / tmax;
    int done = 0;
    for (int L = 0; L < n_launch; ++L) {
        const int iters = std::min(tmax, inner - done);
        const bool fin = (L == n_launch - 1);
        const int src = (L % 2 == 0) ? 1 : 5, dst = (L % 2 == 0) ? 5 : 1;  // X / Y sets
        for (int g = 0; g < G; ++g) {
            const RowSets r = row_sets(sl[g], W);
            FgpArgs a;
            a.H = H;
            a.W = W;
            a.Ha = sl[g].Hl + 2 * GR; a.grow0 = sl[g].r0 - GR; a.row_lo = GR; a.rows_out = sl[g].Hl;
            a.v = r.a[0];
            a.p_in = r.a[src]; a.q_in = r.a[src + 1];
            a.r_in = L ? r.a[src + 2] : nullptr;
            a.s_in = L ? r.a[src + 3] : nullptr;
            if (fin) {
                a.p_out = sl[g].p; a.q_out = sl[g].q; a.r_out = nullptr; a.s_out = nullptr;
            } else {
                a.p_out = r.a[dst]; a.q_out = r.a[dst + 1];
                a.r_out = r.a[dst + 2]; a.s_out = r.a[dst + 3];
            }
            a.lam = (float)lam;
            a.eta = (float)(1.0 / (8.0 * lam));
            for (int k = 0; k < kFgpMaxT; ++k) a.beta[k] = (k < iters) ? (float)betas[done + k] : 0.f;
            a.n_iter = iters;
            // T iterations make T rings of the region inexact (each iteration's
            // stencil reaches one point in every direction); the final launch's
            // x = v - lam D^T(p, q) needs one ring more
            a.halo = fin ? iters + 1 : iters;
            a.nonneg = nonneg;
            a.final_ = fin ? 1 : 0;
            a.x_out = sl[g].x_out;
            a.xhat = sl[g].xhat;
            a.h = sl[g].h;
            a.pog = pog;
            a.iteration = (long long)iteration;
            a.bad_iter = (long long*)bad_iter;
            const int IW = RW - 2 * a.halo, IH = RH - 2 * a.halo;
            dim3 grid((W + IW - 1) / IW, (sl[g].Hl + IH - 1) / IH);
            PT_CHECK_CUDA(launch_pdl(nonneg ? fgp2d_kernel<RW, RH, STRIP, true>
                                            : fgp2d_kernel<RW, RH, STRIP, false>,
                                     grid, dim3(RW * (RH / STRIP)), 0, st, a));
            PT_CHECK_LAUNCH();
        }
        if (!fin) {
            rc = fgp2d_rows_exchange(sl, G, W, dst, 4, halo, st);
            if (rc) return rc;
        }
        done += iters;
    }
    return PT_OK;
}

int fgp2d_rows_run(const Fgp2Slab* sl, int G, int H, int W, double lam, int inner, int nonneg,
                   float pog, int64_t iteration, int64_t* bad_iter, const RowHalo* halo,
                   cudaStream_t st)
{
    if (inner < 1) {
        set_error("inner_iterations must be >= 1");
        return PT_EINVAL;
    }
    for (int g = 0; g < G; ++g) {
        if (sl[g].Hl < kRowGhost) {
            set_error("a row slab needs at least %d rows", kRowGhost);
            return PT_EINVAL;
        }
    }
    // the whole-image tile choice (launch_tv_prox), so T and tiles match
    if (fgp2d_big(H, W))
        return fgp2d_rows_run_t<64, 64, 8>(sl, G, H, W, lam, inner, nonneg, pog, iteration,
                                           bad_iter, halo,
                                           std::min(fgp2d_tmax(H, W), kRowGhost - 1), st);
    return fgp2d_rows_run_t<32, 32, 8>(sl, G, H, W, lam, inner, nonneg, pog, iteration, bad_iter,
                                       halo, 3, st);  // rows: T <= kRowGhost - 1
}

// ---------------------------------------------------------------------------
// 3D isotropic FGP on a (Z, H, W) volume (slice-stacked geometry, config 3).
// No reference code exists: the 2D algorithm with a
// third forward difference along z and dual step 1/(12 lam).
//
// One fused launch per inner iteration.  State: the duals P_k and the
// momentum duals R_k = P_k + beta_{k-1} (P_k - P_{k-1}), each a set laid out
// [Zl + 2][3][H][W] (the three components of a plane contiguous, one ghost
// plane below and above).  An iteration reads R_k (with halo), P_k and v and
// writes P_{k+1}, R_{k+1}: 52 B per voxel, with u = max(v - lam D^T R_k, 0)
// recomputed on chip.  A CTA owns a TY x TX column of the volume over a run of
// planes and marches it along z: the R / v / P boxes of plane z + NS - 1 are
// in flight (TMA into an NS-stage shared-memory ring, mbarrier completion;
// cp.async when W % 4 != 0) while u of plane z + 1 and the dual step of plane
// z are computed from shared memory.
//
// z-slabs: a rank (or a virtual slab on one device) owns
// planes [z0, z0 + Zl) of Zg; the ghost planes of the R sets and one ghost
// plane of v above hold the neighbours' boundary planes, refreshed by a halo
// exchange after every iteration (fgp3d_run).  Ghost planes on the global
// boundary are zero.
// ---------------------------------------------------------------------------
struct Fgp3Args {
    int Zl, H, W, z0, Zg, zchunk;
    const float* v;     // [Zl][H][W]
    const float* vtop;  // v of global plane z0 + Zl (ghost)
    const float* P;     // P_{k-1}  [Zl + 2][3][H][W]
    const float* R;     // P_k
    float* Pn;          // P_{k+1}
    float* Rn;          // P_{k+2} (two-iteration pass)
    float lam, eta, beta;  // beta = beta_k (momentum of the output)
    float beta_r;          // R_k = P_k + beta_r (P_k - P_{k-1}) formed on chip
    float beta1 = 0.f;     // beta_{k+1} (three-iteration pass: R_{k+2})
    int nonneg;
    // register-column pass on a z-slab: planes -2, -1 / Zl, Zl + 1 come from
    // 2-plane ghost buffers [side][P_k: 2 x 3 planes, P_{k-1}: 2 x 3, v: 2]
    // (fgp3d_ghost_exchange) instead of the sets' one-plane ghosts
    const float* ghost = nullptr;
};

// TMA descriptors of one launch: R_k and P_k as 4D tensors (W, H, 3, Zl + 2),
// v as (W, H, Zl), its ghost plane as (W, H); zero fill outside.
struct Fgp3Maps {
    CUtensorMap R, P, V, Vt;
    CUtensorMap Rg[2], Pg[2], Vg[2];  // column pass on a z-slab: lower / upper ghosts
};

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(bar), "r"(parity));
}
__device__ __forceinline__ void cpa4(uint32_t dst, const float* src, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 4 : 0));
}

// Stage layout of one plane: the P_k box [3][TY+2][TX+8] (rows i0-1 ..,
// columns j0-4 ..), the P_{k-1} box (same shape, at QOFF) and the v box
// [TY+2][TX+8] (same window); R_k is formed on chip ("PQ" form: 40 B per
// voxel of HBM traffic; storing R as a state of its own took 52 B and was
// slower, 15.35 vs 14.1 ms per 256^3 FGP-100).
template <int TX, int TY, int NS>
struct Fgp3Tile {
    static constexpr int NT = TX * TY / 2;      // 2 output rows per thread
    static constexpr int RW = TX + 8, RR = TY + 2, ARR = RR * RW;
    static constexpr int WIN3 = (3 * ARR + 31) & ~31;
    static constexpr int QOFF = WIN3;
    static constexpr int VOFF = 2 * WIN3;
    static constexpr int STAGE = (VOFF + ARR + 31) & ~31;
    static constexpr int NWW = (TY + 1) * (TX + 1);   // u window
    static constexpr int SMEM_FLOATS = NS * STAGE + 2 * NWW;
    static constexpr int TMA_BYTES_RV = 4 * ARR * 4;
    static constexpr int TMA_BYTES_P = 3 * ARR * 4;
};

template <int TX, int TY, int NS, bool TMA>
__global__ void __launch_bounds__(TX * TY / 2) fgp3d_iter_kernel(Fgp3Args a,
                                                                 const __grid_constant__ Fgp3Maps m)
{
    using T = Fgp3Tile<TX, TY, NS>;
    constexpr int NT = T::NT, RW = T::RW, RR = T::RR, ARR = T::ARR, NWW = T::NWW;
    constexpr int KU = (NWW + NT - 1) / NT;
    extern __shared__ __align__(128) float fsm[];
    __shared__ __align__(8) uint64_t mbar[NS];
    float* sU = fsm + NS * T::STAGE;  // [2][TY+1][TX+1]
    const uint32_t fsm_u32 = (uint32_t)__cvta_generic_to_shared(fsm);

    const int tid = threadIdx.x;
    const int i0 = blockIdx.y * TY, j0 = blockIdx.x * TX;
    const int zb = blockIdx.z * a.zchunk;
    const int ze = min(a.Zl, zb + a.zchunk);
    const int H = a.H, W = a.W;
    const size_t HW = (size_t)H * W;

    if (TMA) {
        if (tid == 0) {
            for (int k = 0; k < NS; ++k)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(&mbar[k])));
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
        __syncthreads();
    }
    pdl_wait<PDL_FGP3D>();  // the dual sets are the predecessor's output
    // plane p (local; -1 / Zl are ghosts) into stage s
    auto stage = [&](int p, int s) {
        const uint32_t sb = fsm_u32 + (uint32_t)(s * T::STAGE) * 4u;
        const bool withv = p >= 0;  // v of plane -1 is never used
        if (TMA) {
            if (tid != 0) return;
            const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&mbar[s]);
            const uint32_t bytes = (uint32_t)((withv ? T::TMA_BYTES_RV : 3 * ARR * 4) + T::TMA_BYTES_P);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"(bytes));
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sb),
                "l"(&m.R), "r"(j0 - 4), "r"(i0 - 1), "r"(0), "r"(p + 1), "r"(bar) : "memory");
            asm volatile(  // P_{k-1} window
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sb + (uint32_t)T::QOFF * 4u),
                "l"(&m.P), "r"(j0 - 4), "r"(i0 - 1), "r"(0), "r"(p + 1), "r"(bar) : "memory");
            if (withv && p < a.Zl)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sb + (uint32_t)T::VOFF * 4u),
                    "l"(&m.V), "r"(j0 - 4), "r"(i0 - 1), "r"(p), "r"(bar) : "memory");
            else if (withv)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3}], [%4];" ::"r"(sb + (uint32_t)T::VOFF * 4u),
                    "l"(&m.Vt), "r"(j0 - 4), "r"(i0 - 1), "r"(bar) : "memory");
        } else {
            // element copies of the used windows (columns j0-1 .. j0+TX, zero fill)
            const size_t b0 = ((size_t)(p + 1) * 3) * HW;
            const float* vb = (p < a.Zl) ? a.v + (size_t)max(p, 0) * HW : a.vtop;
            constexpr int CW = TX + 2, NR = 4 * RR * CW;  // R (3) + v windows
            for (int idx = tid; idx < NR; idx += NT) {
                const int arr = idx / (RR * CW), rem = idx - arr * (RR * CW);
                const int r = rem / CW, c = rem - r * CW;
                const int gi = i0 - 1 + r, gj = j0 - 1 + c;
                const bool ok = gi >= 0 && gi < H && gj >= 0 && gj < W && (arr < 3 || withv);
                const float* src = arr < 3 ? a.R + b0 + arr * HW : vb;
                cpa4(sb + (uint32_t)((arr < 3 ? arr * ARR : T::VOFF) + r * RW + 3 + c) * 4u,
                     src + (ok ? gi * W + gj : 0), ok);
            }
            constexpr int NQ = 3 * RR * CW;  // P_{k-1} windows
            for (int idx = tid; idx < NQ; idx += NT) {
                const int arr = idx / (RR * CW), rem = idx - arr * (RR * CW);
                const int r = rem / CW, c = rem - r * CW;
                const int gi = i0 - 1 + r, gj = j0 - 1 + c;
                const bool ok = gi >= 0 && gi < H && gj >= 0 && gj < W;
                cpa4(sb + (uint32_t)(T::QOFF + arr * ARR + r * RW + 3 + c) * 4u,
                     a.P + b0 + arr * HW + (ok ? gi * W + gj : 0), ok);
            }
            asm volatile("cp.async.commit_group;");
        }
    };
    auto issue = [&](int p) {  // plane p into stage (p - zb + 1) mod NS, if used by this run
        if (p <= a.Zl && p <= ze) stage(p, (p - zb + 1) % NS);
        else if (!TMA) asm volatile("cp.async.commit_group;");
    };
    auto landed = [&](int p) {
        if (TMA) {
            const int u = p - zb + 1;
            mbar_wait((uint32_t)__cvta_generic_to_shared(&mbar[u % NS]), (uint32_t)((u / NS) & 1));
        }
    };
    // this thread's u positions in the (TY+1) x (TX+1) window: staged offset
    // and guard bits (0: i < H-1, 1: i > 0, 2: j < W-1, 3: j > 0, 4: inside)
    int uOff[KU], uG[KU];
#pragma unroll
    for (int k = 0; k < KU; ++k) {
        const int idx = tid + k * NT, r = idx / (TX + 1), c = idx - r * (TX + 1);
        const int gi = i0 + r, gj = j0 + c;
        uOff[k] = (r + 1) * RW + 4 + c;
        uG[k] = (idx < NWW) ? ((gi < H - 1) | ((gi > 0) << 1) | ((gj < W - 1) << 2) |
                               ((gj > 0) << 3) | ((gi < H && gj < W) << 4))
                            : -1;
    }
    // R_k at staged offset o, formed from P_k and P_{k-1}
    const float br = a.beta_r;
    auto rv = [&](const float* st, int o) -> float {
        const float pv = st[o];
        return pv + br * (pv - st[T::QOFF + o]);
    };
    // u of plane z (its stage s) into sU[z & 1]; R_w of z - 1 from stage s1
    auto compute_U = [&](int z, int s, int s1) {
        const int zg = a.z0 + z;
        const bool zlo = zg > 0, zhi = zg < a.Zg - 1;
        const float* st = fsm + s * T::STAGE;
        const float* st1 = fsm + s1 * T::STAGE;
        float* U = sU + (z & 1) * NWW;
#pragma unroll
        for (int k = 0; k < KU; ++k) {
            const int gd = uG[k];
            if (gd < 0) continue;
            const int o = uOff[k];
            float u = 0.f;
            if (gd & 16) {
                // D^T(R) in the order of the reference's _diff_adjoint (+ z)
                float x = (gd & 1) ? -rv(st, o) : 0.f;
                if (gd & 2) x += rv(st, o - RW);
                if (gd & 4) x -= rv(st, ARR + o);
                if (gd & 8) x += rv(st, ARR + o - 1);
                if (zhi) x -= rv(st, 2 * ARR + o);
                if (zlo) x += rv(st1, 2 * ARR + o);
                u = st[T::VOFF + o] - a.lam * x;
                if (a.nonneg) u = (u < 0.f) ? 0.f : u;
            }
            U[tid + k * NT] = u;
        }
    };

    // prologue: planes zb - 1 .. zb + NS - 2 issued; u of zb
    for (int p = zb - 1; p <= zb + NS - 2; ++p) issue(p);
    if (!TMA) asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2));
    landed(zb - 1);
    landed(zb);
    __syncthreads();
    compute_U(zb, 1 % NS, 0);
    const int tx = tid % TX, ty = tid / TX;
    constexpr int RSTEP = TY / 2;
    const int gj = j0 + tx;
    for (int z = zb; z < ze; ++z) {
        const int s0 = (z - zb + 1) % NS, s1 = (z - zb + 2) % NS;  // stages of z, z + 1
        const int zg = a.z0 + z;
        const bool top = zg < a.Zg - 1;
        __syncthreads();      // the stage of plane z - 1 is consumed
        issue(z + NS - 1);    // into it
        if (!TMA) asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2));
        landed(z + 1);
        __syncthreads();
        if (top) compute_U(z + 1, s1, s0);
        __syncthreads();
        const float* st = fsm + s0 * T::STAGE;
        const float* U0 = sU + (z & 1) * NWW;
        const float* U1 = sU + ((z + 1) & 1) * NWW;
        float* __restrict__ pn = a.Pn + ((size_t)(z + 1) * 3) * HW;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int r = ty + rr * RSTEP, gi = i0 + r;
            if (gi >= H || gj >= W) continue;
            const int wi = r * (TX + 1) + tx;
            const int o = (r + 1) * RW + 4 + tx;
            const float uo = U0[wi];
            const float gv = (gi < H - 1) ? U0[wi + TX + 1] - uo : 0.f;
            const float gh = (gj < W - 1) ? U0[wi + 1] - uo : 0.f;
            const float gz = top ? U1[wi] - uo : 0.f;
            const float ph = rv(st, o) + a.eta * gv;
            const float qh = rv(st, ARR + o) + a.eta * gh;
            const float wh = rv(st, 2 * ARR + o) + a.eta * gz;
            const float n2 = fmaf(wh, wh, fmaf(qh, qh, __fmul_rn(ph, ph)));  // pinned order (all 3D paths)
            const float inv = (n2 > 1.f) ? rsqrt_ftz(n2) : 1.f;
            const float p0 = ph * inv, p1 = qh * inv, p2 = wh * inv;
            const int g = gi * W + gj;
            pn[g] = p0;
            pn[HW + g] = p1;
            pn[2 * HW + g] = p2;
        }
    }
    if (!TMA) asm volatile("cp.async.wait_group 0;");
    pdl_trigger<PDL_FGP3D>();
}

__device__ __forceinline__ f2 ld2s(const float* p)
{
    const float2 v = *reinterpret_cast<const float2*>(p);
    return pk(v.x, v.y);
}
__device__ __forceinline__ void st2s(float* p, f2 v)
{
    float2 w;
    upk(v, w.x, w.y);
    *reinterpret_cast<float2*>(p) = w;
}
// (n2 > 1 ? rsqrt(n2) : 1) per lane
__device__ __forceinline__ f2 inv_norm2(f2 n2)
{
    float a, b;
    upk(n2, a, b);
    return pk((a > 1.f) ? rsqrt_ftz(a) : 1.f, (b > 1.f) ? rsqrt_ftz(b) : 1.f);
}

// caller duals (three [Zl][H][W] arrays) -> interiors of the P and R sets
__global__ void fgp3d_pack_kernel(const float* p, const float* q, const float* w, float* pset,
                                  float* rset, int Zl, int H, int W)
{
    const size_t HW = (size_t)H * W, n = (size_t)Zl * HW;
    for (size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
         o += (size_t)gridDim.x * blockDim.x) {
        const size_t z = o / HW, ij = o - z * HW;
        const size_t d = ((z + 1) * 3) * HW + ij;
        const float a = p[o], b = q[o], c = w[o];
        pset[d] = a; pset[d + HW] = b; pset[d + 2 * HW] = c;
        rset[d] = a; rset[d + HW] = b; rset[d + 2 * HW] = c;
    }
}

// x = max(v - lam D^T(P), 0), h += (p/gamma)(x - x_hat), duals back to the caller
__global__ void fgp3d_final_kernel(Fgp3Args a, float* p_out, float* q_out, float* w_out,
                                   float* x_out, const float* xhat, float* h, float pog,
                                   long long iteration, long long* bad_iter)
{
    pdl_wait();
    const int H = a.H, W = a.W;
    const size_t HW = (size_t)H * W, n = (size_t)a.Zl * HW;
    for (size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
         o += (size_t)gridDim.x * blockDim.x) {
        const int z = (int)(o / HW);
        const size_t ij = o - (size_t)z * HW;
        const int i = (int)(ij / W), j = (int)(ij - (size_t)i * W);
        const int zg = a.z0 + z;
        const float* P = a.P + ((size_t)(z + 1) * 3) * HW + ij;
        const float pc = P[0], qc = P[HW], wc = P[2 * HW];
        float x = (i < H - 1) ? -pc : 0.f;
        if (i > 0) x += P[-(ptrdiff_t)W];
        if (j < W - 1) x -= qc;
        if (j > 0) x += P[HW - 1];
        if (zg < a.Zg - 1) x -= wc;
        if (zg > 0) x += P[2 * HW - 3 * (ptrdiff_t)HW];
        float xv = a.v[o] - a.lam * x;
        if (a.nonneg) xv = (xv < 0.f) ? 0.f : xv;
        x_out[o] = xv;
        if (h) h[o] = h[o] + pog * (xv - xhat[o]);
        p_out[o] = pc;
        q_out[o] = qc;
        w_out[o] = wc;
        if (!isfinite(xv) && bad_iter) atomicMin(bad_iter, iteration);
    }
    pdl_trigger();
}

// Ghost buffers of the multi-iteration passes on z-slabs: per side up to
// kGhostD planes of P_k (3 components each), of P_{k-1} and of v; a pass with
// D <= kGhostD iterations uses the first D plane slots of each region.
constexpr int kGhostD = 3;
constexpr int kGhostSide = 7 * kGhostD;  // planes per side
constexpr int kGhostPm = 3 * kGhostD;    // P_{k-1} region (planes from the side start)
constexpr int kGhostV = 6 * kGhostD;     // v region

int64_t fgp3d_slab_floats(int Zl, int H, int W)
{
    // four sets (P, R ping-pong) + the ghost plane of v + the column passes'
    // ghosts (2 sides x kGhostSide planes)
    return 12 * (int64_t)(Zl + 2) * H * W + (int64_t)H * W + 2 * kGhostSide * (int64_t)H * W;
}
static inline float* fgp3d_ghost(float* work, int side, int Zl, int H, int W)
{
    return work + 12 * (size_t)(Zl + 2) * H * W + (size_t)H * W +
           (size_t)side * kGhostSide * H * W;
}

// set k of a slab workspace: 0 / 1 = P, R of the even iterations, 2 / 3 = odd
static inline float* fgp3d_set(float* work, int which, int Zl, int H, int W)
{
    return work + (size_t)which * 3 * (size_t)(Zl + 2) * H * W;
}
static inline float* fgp3d_vtop(float* work, int Zl, int H, int W)
{
    return work + 12 * (size_t)(Zl + 2) * H * W;
}

// Ghost planes of set `which` (and of v when `with_v`) for every local slab:
// neighbours inside the process by copies, across ranks by the halo callback
// (NCCL send/recv with rank -+ 1).
static int fgp3d_exchange(const Fgp3Slab* sl, int G, int H, int W, int which, bool with_v,
                          const ZHalo* halo, cudaStream_t st)
{
    const size_t HW = (size_t)H * W, plane3 = 3 * HW;
    for (int g = 0; g < G; ++g) {
        float* set = fgp3d_set(sl[g].work, which, sl[g].Zl, H, W);
        if (g > 0) {
            const float* lo = fgp3d_set(sl[g - 1].work, which, sl[g - 1].Zl, H, W);
            PT_CHECK_CUDA(cudaMemcpyAsync(set, lo + (size_t)sl[g - 1].Zl * plane3, plane3 * 4,
                                          cudaMemcpyDeviceToDevice, st));
        }
        if (g + 1 < G) {
            const float* hi = fgp3d_set(sl[g + 1].work, which, sl[g + 1].Zl, H, W);
            PT_CHECK_CUDA(cudaMemcpyAsync(set + (size_t)(sl[g].Zl + 1) * plane3, hi + plane3,
                                          plane3 * 4, cudaMemcpyDeviceToDevice, st));
            if (with_v)
                PT_CHECK_CUDA(cudaMemcpyAsync(fgp3d_vtop(sl[g].work, sl[g].Zl, H, W), sl[g + 1].v,
                                              HW * 4, cudaMemcpyDeviceToDevice, st));
        }
    }
    if (halo && halo->world > 1) {
        // remote neighbours of the first / last local slab
        const Fgp3Slab& f = sl[0];
        const Fgp3Slab& l = sl[G - 1];
        float* fs = fgp3d_set(f.work, which, f.Zl, H, W);
        float* ls = fgp3d_set(l.work, which, l.Zl, H, W);
        int rc = halo->exchange(halo->ctx, fs + plane3, fs, ls + (size_t)l.Zl * plane3,
                                ls + (size_t)(l.Zl + 1) * plane3, plane3, st);
        if (rc) return rc;
        if (with_v) {
            rc = halo->exchange(halo->ctx, f.v, nullptr, nullptr, fgp3d_vtop(l.work, l.Zl, H, W),
                                HW, st);
            if (rc) return rc;
        }
    }
    return PT_OK;
}

// The column pass's 2-plane ghosts of z-slab g: its lower buffer receives the
// two top planes of slab g - 1, its upper buffer the two bottom planes of
// slab g + 1, for the sets of P_k and P_{k-1} (and for v when with_v), by
// device copies between local slabs and the halo callback (ncclSend /
// ncclRecv) between ranks.  Buffers on the global boundary stay zero.
static int fgp3d_ghost_exchange(const Fgp3Slab* sl, int G, int H, int W, int set_k, int set_m,
                                bool with_v, const ZHalo* halo, cudaStream_t st, int D = 2)
{
    const size_t HW = (size_t)H * W, plane3 = 3 * HW;
    // (source of the D planes [lo, lo + D) of slab g, offset in a ghost side, count)
    struct Arr { int kind; size_t goff, count; };  // kind 0: set k, 1: set m, 2: v
    const Arr arrs[3] = {{0, 0, D * plane3}, {1, kGhostPm * HW, D * plane3},
                         {2, kGhostV * HW, D * HW}};
    auto src = [&](const Fgp3Slab& q, const Arr& ar, bool top) -> const float* {
        if (ar.kind == 2) return q.v + (top ? (size_t)(q.Zl - D) * HW : 0);
        const float* set = fgp3d_set(q.work, ar.kind == 0 ? set_k : set_m, q.Zl, H, W);
        return set + (top ? (size_t)(q.Zl - D + 1) * plane3 : plane3);  // set index = plane + 1
    };
    for (const Arr& ar : arrs) {
        if (ar.kind == 2 && !with_v) continue;
        for (int g = 0; g < G; ++g) {
            float* lo = fgp3d_ghost(sl[g].work, 0, sl[g].Zl, H, W) + ar.goff;
            float* hi = fgp3d_ghost(sl[g].work, 1, sl[g].Zl, H, W) + ar.goff;
            if (g > 0)
                PT_CHECK_CUDA(cudaMemcpyAsync(lo, src(sl[g - 1], ar, true), ar.count * 4,
                                              cudaMemcpyDeviceToDevice, st));
            if (g + 1 < G)
                PT_CHECK_CUDA(cudaMemcpyAsync(hi, src(sl[g + 1], ar, false), ar.count * 4,
                                              cudaMemcpyDeviceToDevice, st));
        }
        if (halo && halo->world > 1) {
            const Fgp3Slab& f = sl[0];
            const Fgp3Slab& l = sl[G - 1];
            const int rc = halo->exchange(
                halo->ctx, src(f, ar, false), fgp3d_ghost(f.work, 0, f.Zl, H, W) + ar.goff,
                src(l, ar, true), fgp3d_ghost(l.work, 1, l.Zl, H, W) + ar.goff, ar.count, st);
            if (rc) return rc;
        }
    }
    return PT_OK;
}

template <int TX, int TY, int NS, bool TMA>
static int fgp3d_launch(Fgp3Args& a, int sm_count, cudaStream_t st)
{
    using T = Fgp3Tile<TX, TY, NS>;
    const size_t smem = (size_t)T::SMEM_FLOATS * 4;
    {
        const int rc = ensure_smem((const void*)fgp3d_iter_kernel<TX, TY, NS, TMA>, smem);
        if (rc) return rc;
    }
    Fgp3Maps m;
    memset(&m, 0, sizeof(m));
    if (TMA) {
        const cuuint64_t W = a.W, H = a.H;
        const cuuint64_t d4[4] = {W, H, 3, (cuuint64_t)a.Zl + 2};
        const cuuint32_t bR[4] = {(cuuint32_t)T::RW, (cuuint32_t)T::RR, 3, 1};
        const cuuint64_t d3[3] = {W, H, (cuuint64_t)a.Zl};
        const cuuint32_t b3[3] = {(cuuint32_t)T::RW, (cuuint32_t)T::RR, 1};
        int rc = make_map(&m.R, a.R, 4, d4, bR);
        if (!rc) rc = make_map(&m.P, a.P, 4, d4, bR);
        if (!rc) rc = make_map(&m.V, a.v, 3, d3, b3);
        if (!rc) rc = make_map(&m.Vt, a.vtop, 2, d3, b3);
        if (rc) return rc;
    }
    static const int zc_env = [] {
        const char* e = getenv("PT_FGP3_ZCHUNK");
        return e ? std::max(0, atoi(e)) : 0;  // 0 / empty: the default
    }();
    const int gx = (a.W + TX - 1) / TX, gy = (a.H + TY - 1) / TY;
    // runs of 16 planes (two extra staged planes per run); measured at 256^3:
    // 8 -> 155 us, 16 -> 153 us, 32 -> 165 us, 64 -> 189 us per iteration
    a.zchunk = zc_env ? zc_env : 16;
    dim3 grid(gx, gy, (a.Zl + a.zchunk - 1) / a.zchunk);
    PT_CHECK_CUDA(launch_pdl(fgp3d_iter_kernel<TX, TY, NS, TMA>, grid, dim3(T::NT), smem, st, a,
                             m));
    PT_CHECK_LAUNCH();
    return PT_OK;
}

// ---------------------------------------------------------------------------
// Two inner iterations per HBM pass, register-column form (single slab, TMA,
// PQ).  A thread owns two x-adjacent columns (f32x2 math) of a BY x 2*BX2
// tile (the core minus a 2-point ring that the two iterations make inexact)
// and marches them along z; its columns' values live in registers, only the
// stencil's in-plane neighbours cross threads (R_y / R_x of the point above /
// left, u of the point below / right) through shared-memory planes that are
// double-buffered by step parity, so ONE barrier per plane step serves both
// iterations.  The iterations run as lagged phases: at step s phase 0 turns
// the staged P_k, P_{k-1}, v of plane s + 1 into u_k(s + 1) and P_{k+1}(s) and
// hands R_{k+1}(s) to phase 1 in registers; phase 1 turns it into
// u_{k+1}(s - 1) and P_{k+2}(s - 2).  Inputs arrive by TMA (one box per array
// and plane, 16-byte aligned origin, zero fill off the volume) into a 3-stage
// ring.  Tiles strictly inside the image skip every guard.  Every value is
// the one-iteration kernel's expression in its operation order, so the pass
// is bitwise equal to two fgp3d_iter_kernel launches.
// ---------------------------------------------------------------------------
template <int BX2, int BY, int NS_ = 3>
struct Fgp3Col {
    static constexpr int NT = BX2 * BY;
    static constexpr int BXP = 2 * BX2;       // tile width in points
    static constexpr int NS = NS_;            // TMA ring stages (planes)
    static constexpr int BW = BXP + 4;        // staged box width (origin two points left)
    static constexpr int PL = BW * BY;        // one staged array plane (floats)
    static constexpr int STAGE = 7 * PL;      // P_k (3), P_{k-1} (3), v
    static constexpr int XPL = 2 * (NT + 1);  // exchange plane: float2 per thread + zero slot
    static constexpr int XR = NS * STAGE;     // [2 parity][R_y0, R_x0, R_y1, R_x1][XPL]
    static constexpr int XU = XR + 8 * XPL;   // [2 parity][u0, u1][XPL]
    static constexpr int SMEM_FLOATS = XU + 4 * XPL;
    static constexpr uint32_t TMA_BYTES = (uint32_t)STAGE * 4u;
    static constexpr int CX = BXP - 4, CY = BY - 4;  // exact core (two rings)
    static_assert(CX % 4 == 0, "16-byte aligned tile origins (TMA)");
    static_assert((STAGE * 4) % 128 == 0 && (PL * 4) % 128 == 0, "128-byte aligned TMA boxes");
};

__device__ __forceinline__ f2 ldx2(const float* p) { return ld2s(p); }
// per-lane select (lanes a / b)
__device__ __forceinline__ f2 sel2(bool ca, bool cb, f2 x, f2 y)
{
    float xa, xb, ya, yb;
    upk(x, xa, xb);
    upk(y, ya, yb);
    return pk(ca ? xa : ya, cb ? xb : yb);
}

template <int BX2, int BY, int MINB, int NS = 3>
__global__ void __launch_bounds__(BX2 * BY, MINB)
    fgp3d_col_kernel(Fgp3Args a, const __grid_constant__ Fgp3Maps m)
{
    using T = Fgp3Col<BX2, BY, NS>;
    constexpr int NT = T::NT, XPL = T::XPL;
    extern __shared__ __align__(128) float fsm[];
    __shared__ __align__(8) uint64_t mbar[T::NS];
    const int tid = threadIdx.x;
    const int tx = tid % BX2, ty = tid / BX2;
    const int j0 = blockIdx.x * T::CX - 2, i0 = blockIdx.y * T::CY - 2;
    const int zb = blockIdx.z * a.zchunk;
    const int ze = min(a.Zl, zb + a.zchunk);
    const int H = a.H, W = a.W;  // W even: a pair is inside or outside the image as a whole
    const size_t HW = (size_t)H * W;
    const int i = i0 + ty, ja = j0 + 2 * tx;
    const bool inimg = i >= 0 && i < H && ja >= 0 && ja < W;
    const bool i_lt = i < H - 1, i_gt = i > 0;
    const bool jgt_a = ja > 0, jlt_b = ja + 1 < W - 1;  // lane b is never at j = 0, lane a never at W - 1
    const bool core = tx >= 1 && tx < BX2 - 1 && ty >= 2 && ty < BY - 2 && inimg;
    // the whole tile and one point around it strictly inside the image: no guards
    const bool interior = i0 >= 1 && i0 + BY <= H - 1 && j0 >= 1 && j0 + T::BXP <= W - 1;
    // neighbour slots (float2 index) of the exchange planes; the zero slot off the tile
    const int n_up = ty > 0 ? tid - BX2 : NT, n_down = ty < BY - 1 ? tid + BX2 : NT;
    const int n_left = tx > 0 ? tid - 1 : NT, n_right = tx < BX2 - 1 ? tid + 1 : NT;
    const int own = ty * T::BW + 2 * tx + 2;  // this pair in a staged plane
    const f2 br2 = pk(a.beta_r, a.beta_r), bk2 = pk(a.beta, a.beta);
    const f2 eta2 = pk(a.eta, a.eta), nlam2 = pk(-a.lam, -a.lam);
    const f2 z2 = pk(0.f, 0.f), nz2 = pk(-0.f, -0.f);
    const bool nonneg = a.nonneg != 0;
    const int Zg = a.Zg;
    const uint32_t fsm_u32 = (uint32_t)__cvta_generic_to_shared(fsm);
    float* XR = fsm + T::XR;
    float* XU = fsm + T::XU;

    if (tid == 0) {
        for (int k = 0; k < T::NS; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&mbar[k])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 12) {  // zero slots of the twelve exchange planes
        float* pl = (tid < 8 ? XR + tid * XPL : XU + (tid - 8) * XPL) + 2 * NT;
        pl[0] = 0.f;
        pl[1] = 0.f;
    }
    __syncthreads();
    pdl_wait<PDL_FGP3D>();  // the dual sets are the predecessor's output
    const int pfirst = zb - 2, plast = ze + 2;  // input planes of this run
    auto issue = [&](int p, int st) {
        const uint32_t sb = fsm_u32 + (uint32_t)(st * T::STAGE) * 4u;
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&mbar[st]);
        // a slab's planes outside [0, Zl) come from its ghost buffers
        const bool gh = a.ghost && (p < 0 || p >= a.Zl);
        const int side = p < 0 ? 0 : 1;
        const CUtensorMap* mr = gh ? &m.Rg[side] : &m.R;
        const CUtensorMap* mp = gh ? &m.Pg[side] : &m.P;
        const CUtensorMap* mv = gh ? &m.Vg[side] : &m.V;
        const int pz = gh ? (p < 0 ? p + 2 : p - a.Zl) : p + 1;  // set / ghost plane index
        const int vz = gh ? pz : p;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(T::TMA_BYTES));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sb),
            "l"(mr), "r"(j0 - 2), "r"(i0), "r"(0), "r"(pz), "r"(bar) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sb + (uint32_t)(3 * T::PL) * 4u),
            "l"(mp), "r"(j0 - 2), "r"(i0), "r"(0), "r"(pz), "r"(bar) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sb + (uint32_t)(6 * T::PL) * 4u),
            "l"(mv), "r"(j0 - 2), "r"(i0), "r"(vz), "r"(bar) : "memory");
    };
    if (tid == 0)
        for (int k = 0; k < T::NS; ++k) issue(pfirst + k, k);

    // carried state (zeros before the run: they only feed planes outside the
    // exact cone of [zb, ze))
    f2 r0p[3] = {z2, z2, z2}, r1p[3] = {z2, z2, z2};  // R_k(s), R_{k+1}(s - 2)
    f2 r1in[3] = {z2, z2, z2};                        // R_{k+1}(s - 1) (handoff)
    f2 u0p = z2, u1p = z2;                            // u_k(s), u_{k+1}(s - 2)
    f2 pk_own[3] = {z2, z2, z2};                      // P_k(s)
    f2 vq0 = z2, vq1 = z2;                            // v(s), v(s - 1)
    const ptrdiff_t plane3 = 3 * (ptrdiff_t)HW;
    const size_t gij = core ? (size_t)i * W + ja : 0;
    float* o1 = a.Pn + plane3 * (zb - 3) + gij;  // P_{k+1}(s): set index s + 1
    float* o2 = a.Rn + plane3 * (zb - 5) + gij;  // P_{k+2}(s - 2): set index s - 1

    // u = clamp(v - lam D^T R) in _diff_adjoint's order (+ z).  XYI: the tile
    // is strictly inside the image (no in-plane guards); ZI: every z guard of
    // the step holds.  Specialised at compile time so the common case has no
    // selects and no predicated merges.
    auto u_of = [&](auto XYI, auto ZI, const f2 (&r)[3], f2 rup, f2 rleft, f2 r2low, f2 v,
                    bool zhi, bool zlo) {
        f2 x;
        if constexpr (decltype(XYI)::value) {
            x = add2(sub2(add2(sub2(nz2, r[0]), rup), r[1]), rleft);
        } else {
            x = i_lt ? sub2(nz2, r[0]) : z2;
            x = i_gt ? add2(x, rup) : x;
            x = sel2(true, jlt_b, sub2(x, r[1]), x);
            x = sel2(jgt_a, true, add2(x, rleft), x);
        }
        if constexpr (decltype(ZI)::value) {
            x = add2(sub2(x, r[2]), r2low);
        } else {
            x = zhi ? sub2(x, r[2]) : x;
            x = zlo ? add2(x, r2low) : x;
        }
        float ua, ub;
        upk(fma2(x, nlam2, v), ua, ub);
        ua = (nonneg && ua < 0.f) ? 0.f : ua;
        ub = (nonneg && ub < 0.f) ? 0.f : ub;
        if constexpr (!decltype(XYI)::value) {
            ua = inimg ? ua : 0.f;
            ub = inimg ? ub : 0.f;
        }
        return pk(ua, ub);
    };
    // the dual step: R + eta D u, projected; zero off the image / volume
    auto dual = [&](auto XYI, auto ZI, const f2 (&r)[3], f2 uo, f2 udown, f2 uright, f2 uz,
                    bool top, bool zlive, f2 (&pn)[3]) {
        f2 gv = sub2(udown, uo), gh = sub2(uright, uo);
        if constexpr (!decltype(XYI)::value) {
            gv = i_lt ? gv : z2;
            gh = sel2(true, jlt_b, gh, z2);
        }
        f2 gz;
        if constexpr (decltype(ZI)::value) gz = sub2(uz, uo);
        else gz = top ? sub2(uz, uo) : z2;
        const f2 ph = fma2(gv, eta2, r[0]);
        const f2 qh = fma2(gh, eta2, r[1]);
        const f2 wh = fma2(gz, eta2, r[2]);
        const f2 inv = inv_norm2(fma2(wh, wh, fma2(qh, qh, mul2(ph, ph))));  // pinned order
        pn[0] = mul2(ph, inv);
        pn[1] = mul2(qh, inv);
        pn[2] = mul2(wh, inv);
        if constexpr (!(decltype(XYI)::value && decltype(ZI)::value)) {
            const bool live = zlive && inimg;
            pn[0] = live ? pn[0] : z2;
            pn[1] = live ? pn[1] : z2;
            pn[2] = live ? pn[2] : z2;
        }
    };

    int stg = 0;         // stage of plane s + 1
    uint32_t phase = 0;  // bit k: parity of stage k's next completion
    // One plane step.  The two-deep shift registers (R_{k+1}: previous /
    // handoff, v: v(s) / v(s - 1)) and the one-deep ones are passed by role,
    // so the loop below alternates roles every step instead of moving values.
    auto step = [&](auto XYI, auto ZI, int s, f2 (&r1_prev)[3], f2 (&r1_in)[3],
                    f2 (&r0_prev)[3], f2 (&r0_cur)[3], f2 (&pk_prev)[3], f2 (&pk_cur)[3],
                    f2& u0_prev, f2& u0_cur, f2& u1_prev, f2& u1_cur, f2& v_m1) {
        const int par = s & 1;
        mbar_wait((uint32_t)__cvta_generic_to_shared(&mbar[stg]), (phase >> stg) & 1u);
        phase ^= 1u << stg;
        const float* sp = fsm + stg * T::STAGE + own;
        const f2 v1 = ldx2(sp + 6 * T::PL);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            pk_cur[c] = ldx2(sp + c * T::PL);
            r0_cur[c] = fma2(sub2(pk_cur[c], ldx2(sp + (3 + c) * T::PL)), br2, pk_cur[c]);  // R_k(s + 1)
        }
        float* xr = XR + par * 4 * XPL;
        st2s(xr + 2 * tid, r0_cur[0]);
        st2s(xr + XPL + 2 * tid, r0_cur[1]);
        st2s(xr + 2 * XPL + 2 * tid, r1_in[0]);
        st2s(xr + 3 * XPL + 2 * tid, r1_in[1]);
        __syncthreads();  // exchange planes of step s written; step s - 1 fully read
        // the stage of plane s (read at step s - 1) takes plane s + NS
        if (tid == 0 && s >= pfirst && s + T::NS <= plast)
            issue(s + T::NS, stg == 0 ? T::NS - 1 : stg - 1);
        stg = stg + 1 == T::NS ? 0 : stg + 1;
        const float* xu_prev = XU + (par ^ 1) * 2 * XPL;
        float* xu = XU + par * 2 * XPL;
        const int z1 = a.z0 + s + 1, z0 = a.z0 + s, zm1 = a.z0 + s - 1, zm2 = a.z0 + s - 2;
        // ---- phase 0: u_k(s + 1), P_{k+1}(s)
        u0_cur = u_of(XYI, ZI, r0_cur, ldx2(xr + 2 * n_up),
                      pk(xr[XPL + 2 * n_left + 1], lo_of(r0_cur[1])), r0_prev[2], v1,
                      z1 < Zg - 1, z1 > 0);
        st2s(xu + 2 * tid, u0_cur);
        f2 p1[3];
        dual(XYI, ZI, r0_prev, u0_prev, ldx2(xu_prev + 2 * n_down),
             pk(hi_of(u0_prev), xu_prev[2 * n_right]), u0_cur, z0 < Zg - 1, z0 >= 0 && z0 < Zg,
             p1);
        // ---- phase 1: u_{k+1}(s - 1), P_{k+2}(s - 2)
        u1_cur = u_of(XYI, ZI, r1_in, ldx2(xr + 2 * XPL + 2 * n_up),
                      pk(xr[3 * XPL + 2 * n_left + 1], lo_of(r1_in[1])), r1_prev[2], v_m1,
                      zm1 < Zg - 1, zm1 > 0);
        st2s(xu + XPL + 2 * tid, u1_cur);
        f2 p2[3];
        dual(XYI, ZI, r1_prev, u1_prev, ldx2(xu_prev + XPL + 2 * n_down),
             pk(hi_of(u1_prev), xu_prev[XPL + 2 * n_right]), u1_cur, zm2 < Zg - 1,
             zm2 >= 0 && zm2 < Zg, p2);
        // ---- outputs of the run's own planes (exact core only)
        o1 += plane3;
        o2 += plane3;
        if (core && s >= zb && s < ze) {
            st2s(o1, p1[0]); st2s(o1 + HW, p1[1]); st2s(o1 + 2 * HW, p1[2]);
        }
        if (core && s - 2 >= zb && s - 2 < ze) {
            st2s(o2, p2[0]); st2s(o2 + HW, p2[1]); st2s(o2 + 2 * HW, p2[2]);
        }
        // R_{k+1}(s) for phase 1 (the R-form expression) takes the slot of
        // R_{k+1}(s - 2), consumed above; v(s + 1) takes v(s - 1)'s
#pragma unroll
        for (int c = 0; c < 3; ++c) r1_prev[c] = fma2(sub2(p1[c], pk_prev[c]), bk2, p1[c]);
        v_m1 = v1;
    };
    // roles: even steps (A) and odd steps (B); steps whose planes s - 2 .. s + 1
    // are all inside [1, Zg - 2] pass every z guard (ZI)
    f2 r0q[3] = {z2, z2, z2}, pkq[3] = {z2, z2, z2};
    f2 u0q = z2, u1q = z2;
    auto march = [&](auto XYI) {
        const std::true_type zi{};
        const std::false_type zg{};
        int s = zb - 3;
        for (; s + 1 <= ze + 1; s += 2) {
            const int g0 = a.z0 + s;
            if (g0 - 2 >= 1 && g0 + 2 <= Zg - 2) {
                step(XYI, zi, s, r1p, r1in, r0p, r0q, pk_own, pkq, u0p, u0q, u1p, u1q, vq1);
                step(XYI, zi, s + 1, r1in, r1p, r0q, r0p, pkq, pk_own, u0q, u0p, u1q, u1p, vq0);
            } else {
                step(XYI, zg, s, r1p, r1in, r0p, r0q, pk_own, pkq, u0p, u0q, u1p, u1q, vq1);
                step(XYI, zg, s + 1, r1in, r1p, r0q, r0p, pkq, pk_own, u0q, u0p, u1q, u1p, vq0);
            }
        }
        if (s <= ze + 1) step(XYI, zg, s, r1p, r1in, r0p, r0q, pk_own, pkq, u0p, u0q, u1p, u1q, vq1);
    };
    if (interior) march(std::true_type{});
    else march(std::false_type{});
    pdl_trigger<PDL_FGP3D>();
}

template <int BX2, int BY, int MINB, int NS = 3>
static int fgp3d_col_launch(Fgp3Args& a, int sm_count, cudaStream_t st)
{
    using T = Fgp3Col<BX2, BY, NS>;
    const size_t smem = (size_t)T::SMEM_FLOATS * 4;
    {
        const int rc = ensure_smem((const void*)fgp3d_col_kernel<BX2, BY, MINB, NS>, smem);
        if (rc) return rc;
    }
    int per_sm = 0;
    PT_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, fgp3d_col_kernel<BX2, BY, MINB, NS>, T::NT, smem));
    Fgp3Maps m;
    memset(&m, 0, sizeof(m));
    const cuuint64_t W = a.W, H = a.H;
    const cuuint64_t d4[4] = {W, H, 3, (cuuint64_t)a.Zl + 2};
    const cuuint32_t b4[4] = {(cuuint32_t)T::BW, (cuuint32_t)BY, 3, 1};
    const cuuint64_t d3[3] = {W, H, (cuuint64_t)a.Zl};
    const cuuint32_t b3[3] = {(cuuint32_t)T::BW, (cuuint32_t)BY, 1};
    int rc = make_map(&m.R, a.R, 4, d4, b4);
    if (!rc) rc = make_map(&m.P, a.P, 4, d4, b4);
    if (!rc) rc = make_map(&m.V, a.v, 3, d3, b3);
    if (a.ghost) {
        const size_t HW = (size_t)a.W * a.H;
        const cuuint64_t g4[4] = {W, H, 3, 2};
        const cuuint64_t g3[3] = {W, H, 2};
        for (int side = 0; side < 2 && !rc; ++side) {
            const float* gb = a.ghost + (size_t)side * kGhostSide * HW;
            rc = make_map(&m.Rg[side], gb, 4, g4, b4);
            if (!rc) rc = make_map(&m.Pg[side], gb + kGhostPm * HW, 4, g4, b4);
            if (!rc) rc = make_map(&m.Vg[side], gb + kGhostV * HW, 3, g3, b3);
        }
    }
    if (rc) return rc;
    static const int zc_env = [] {
        const char* e = getenv("PT_FGP3_ZCHUNK");
        return e ? std::max(0, atoi(e)) : 0;
    }();
    const int tiles = ((a.W + T::CX - 1) / T::CX) * ((a.H + T::CY - 1) / T::CY);
    // z-runs: each re-marches 5 planes; as few runs as fill whole waves
    int zc = zc_env;
    if (!zc) {
        const int slots = sm_count * std::max(1, per_sm);
        int best_cost = INT32_MAX;
        zc = a.Zl;
        for (int c = 1; c <= std::max(1, a.Zl / 8); ++c) {
            const int run = (a.Zl + c - 1) / c;
            const int waves = (tiles * c + slots - 1) / slots;
            const int cost = waves * (run + 5);
            if (cost < best_cost) { best_cost = cost; zc = run; }
        }
    }
    a.zchunk = zc;
    const dim3 grid((a.W + T::CX - 1) / T::CX, (a.H + T::CY - 1) / T::CY,
                    (a.Zl + a.zchunk - 1) / a.zchunk);
    PT_CHECK_CUDA(launch_pdl(fgp3d_col_kernel<BX2, BY, MINB, NS>, grid, dim3(T::NT), smem, st, a, m));
    PT_CHECK_LAUNCH();
    return PT_OK;
}

// ---------------------------------------------------------------------------
// Three inner iterations per HBM pass (one slab holding the whole volume):
// fgp3d_col_kernel with a third lagged phase.  At step s phase 0 turns the
// staged P_k, P_{k-1}, v of plane s + 1 into u_k(s + 1) and P_{k+1}(s),
// phase 1 turns R_{k+1}(s - 1) into u_{k+1}(s - 1) and P_{k+2}(s - 2), phase 2
// turns R_{k+2}(s - 3) into u_{k+2}(s - 3) and P_{k+3}(s - 4); the next pass
// reads {P_{k+2}, P_{k+3}} as its {P_{k-1}, P_k}.  R_{k+2} needs P_{k+1} two
// planes back (a two-step register delay), phase 2 needs v three planes back.
// Three iterations make a 3-point ring of the tile inexact; the tile origin
// keeps 4 columns on the left so that boxes and point pairs stay aligned
// (16-byte TMA origins, 8-byte pair loads): a 32 x 32-point tile has a
// 24 x 26 exact core.  Every value is the one-iteration kernel's expression
// in its operation order (the same u_of / dual as the two-iteration pass), so
// the pass is bitwise equal to three fgp3d_iter_kernel launches.
// ---------------------------------------------------------------------------
template <int BX2, int BY, int NS_ = 3>
struct Fgp3Col3 {
    static constexpr int NT = BX2 * BY;
    static constexpr int BXP = 2 * BX2;       // tile width in points (= box width)
    static constexpr int NS = NS_;            // TMA ring stages (planes)
    static constexpr int BW = BXP;            // staged box: the tile itself
    static constexpr int PL = BW * BY;        // one staged array plane (floats)
    static constexpr int STAGE = 7 * PL;      // P_k (3), P_{k-1} (3), v
    static constexpr int XPL = 2 * (NT + 1);  // exchange plane: float2 per thread + zero slot
    static constexpr int XR = NS * STAGE;     // [2 parity][R_y, R_x of phases 0, 1, 2][XPL]
    static constexpr int XU = XR + 12 * XPL;  // [2 parity][u of phases 0, 1, 2][XPL]
    static constexpr int SMEM_FLOATS = XU + 6 * XPL;
    static constexpr uint32_t TMA_BYTES = (uint32_t)STAGE * 4u;
    static constexpr int CX = BXP - 8, CY = BY - 6;  // exact core
    static_assert(CX % 4 == 0 && BW % 4 == 0, "16-byte aligned tile origins (TMA)");
    static_assert((STAGE * 4) % 128 == 0 && (PL * 4) % 128 == 0, "128-byte aligned TMA boxes");
};

template <int BX2, int BY, int NS = 3>
__global__ void __launch_bounds__(BX2 * BY, 1)
    fgp3d_col3_kernel(Fgp3Args a, const __grid_constant__ Fgp3Maps m)
{
    using T = Fgp3Col3<BX2, BY, NS>;
    constexpr int NT = T::NT, XPL = T::XPL;
    extern __shared__ __align__(128) float fsm[];
    __shared__ __align__(8) uint64_t mbar[T::NS];
    const int tid = threadIdx.x;
    const int tx = tid % BX2, ty = tid / BX2;
    const int j0 = blockIdx.x * T::CX - 4, i0 = blockIdx.y * T::CY - 3;
    const int zb = blockIdx.z * a.zchunk;
    const int ze = min(a.Zl, zb + a.zchunk);
    const int H = a.H, W = a.W;  // W even: a pair is inside or outside the image as a whole
    const size_t HW = (size_t)H * W;
    const int i = i0 + ty, ja = j0 + 2 * tx;
    const bool inimg = i >= 0 && i < H && ja >= 0 && ja < W;
    const bool i_lt = i < H - 1, i_gt = i > 0;
    const bool jgt_a = ja > 0, jlt_b = ja + 1 < W - 1;
    const bool core = tx >= 2 && tx < BX2 - 2 && ty >= 3 && ty < BY - 3 && inimg;
    const bool interior = i0 >= 1 && i0 + BY <= H - 1 && j0 >= 1 && j0 + T::BXP <= W - 1;
    const int n_up = ty > 0 ? tid - BX2 : NT, n_down = ty < BY - 1 ? tid + BX2 : NT;
    const int n_left = tx > 0 ? tid - 1 : NT, n_right = tx < BX2 - 1 ? tid + 1 : NT;
    const int own = ty * T::BW + 2 * tx;  // this pair in a staged plane
    const f2 br2 = pk(a.beta_r, a.beta_r), bk2 = pk(a.beta, a.beta), bk12 = pk(a.beta1, a.beta1);
    const f2 eta2 = pk(a.eta, a.eta), nlam2 = pk(-a.lam, -a.lam);
    const f2 z2 = pk(0.f, 0.f), nz2 = pk(-0.f, -0.f);
    const bool nonneg = a.nonneg != 0;
    const int Zg = a.Zg;
    const uint32_t fsm_u32 = (uint32_t)__cvta_generic_to_shared(fsm);
    float* XR = fsm + T::XR;
    float* XU = fsm + T::XU;

    if (tid == 0) {
        for (int k = 0; k < T::NS; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&mbar[k])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 18) {  // zero slots of the eighteen exchange planes
        float* pl = (tid < 12 ? XR + tid * XPL : XU + (tid - 12) * XPL) + 2 * NT;
        pl[0] = 0.f;
        pl[1] = 0.f;
    }
    __syncthreads();
    pdl_wait<PDL_FGP3D>();  // the dual sets are the predecessor's output
    const int pfirst = zb - 3, plast = ze + 4;  // input planes of this run
    auto issue = [&](int p, int st) {
        const uint32_t sb = fsm_u32 + (uint32_t)(st * T::STAGE) * 4u;
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&mbar[st]);
        // a slab's planes outside [0, Zl) come from its 3-plane ghost buffers;
        // planes outside the volume: the sets' zero ghost planes, or zero fill
        const bool gh = a.ghost && (p < 0 || p >= a.Zl);
        const int side = p < 0 ? 0 : 1;
        const CUtensorMap* mr = gh ? &m.Rg[side] : &m.R;
        const CUtensorMap* mp = gh ? &m.Pg[side] : &m.P;
        const CUtensorMap* mv = gh ? &m.Vg[side] : &m.V;
        const int pz = gh ? (p < 0 ? p + 3 : p - a.Zl) : p + 1;  // set / ghost plane index
        const int vz = gh ? pz : p;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(T::TMA_BYTES));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sb),
            "l"(mr), "r"(j0), "r"(i0), "r"(0), "r"(pz), "r"(bar) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sb + (uint32_t)(3 * T::PL) * 4u),
            "l"(mp), "r"(j0), "r"(i0), "r"(0), "r"(pz), "r"(bar) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sb + (uint32_t)(6 * T::PL) * 4u),
            "l"(mv), "r"(j0), "r"(i0), "r"(vz), "r"(bar) : "memory");
    };
    if (tid == 0)
        for (int k = 0; k < T::NS; ++k) issue(pfirst + k, k);

    // carried state (zeros before the run: they only feed planes outside the
    // exact cone of [zb, ze))
    f2 r0a[3] = {z2, z2, z2}, r0b[3] = {z2, z2, z2};  // R_k(s), R_k(s + 1)
    f2 r1a[3] = {z2, z2, z2}, r1b[3] = {z2, z2, z2};  // R_{k+1}(s - 2), R_{k+1}(s - 1)
    f2 r2a[3] = {z2, z2, z2}, r2b[3] = {z2, z2, z2};  // R_{k+2}(s - 4), R_{k+2}(s - 3)
    f2 pka[3] = {z2, z2, z2}, pkb[3] = {z2, z2, z2};  // P_k(s), P_k(s + 1)
    f2 pda[3] = {z2, z2, z2}, pdb[3] = {z2, z2, z2};  // P_{k+1} two steps back (by parity)
    f2 u0a = z2, u0b = z2, u1a = z2, u1b = z2, u2a = z2, u2b = z2;
    f2 va = z2, vb = z2, wa = z2, wb = z2;            // v(s - 1), v(s - 3) (by parity)
    const ptrdiff_t plane3 = 3 * (ptrdiff_t)HW;
    const size_t gij = core ? (size_t)i * W + ja : 0;
    float* o2 = a.Pn + plane3 * (zb - 6) + gij;  // P_{k+2}(s - 2): set index s - 1
    float* o3 = a.Rn + plane3 * (zb - 8) + gij;  // P_{k+3}(s - 4): set index s - 3

    auto u_of = [&](auto XYI, auto ZI, const f2 (&r)[3], f2 rup, f2 rleft, f2 r2low, f2 v,
                    bool zhi, bool zlo) {
        f2 x;
        if constexpr (decltype(XYI)::value) {
            x = add2(sub2(add2(sub2(nz2, r[0]), rup), r[1]), rleft);
        } else {
            x = i_lt ? sub2(nz2, r[0]) : z2;
            x = i_gt ? add2(x, rup) : x;
            x = sel2(true, jlt_b, sub2(x, r[1]), x);
            x = sel2(jgt_a, true, add2(x, rleft), x);
        }
        if constexpr (decltype(ZI)::value) {
            x = add2(sub2(x, r[2]), r2low);
        } else {
            x = zhi ? sub2(x, r[2]) : x;
            x = zlo ? add2(x, r2low) : x;
        }
        float ua, ub;
        upk(fma2(x, nlam2, v), ua, ub);
        ua = (nonneg && ua < 0.f) ? 0.f : ua;
        ub = (nonneg && ub < 0.f) ? 0.f : ub;
        if constexpr (!decltype(XYI)::value) {
            ua = inimg ? ua : 0.f;
            ub = inimg ? ub : 0.f;
        }
        return pk(ua, ub);
    };
    auto dual = [&](auto XYI, auto ZI, const f2 (&r)[3], f2 uo, f2 udown, f2 uright, f2 uz,
                    bool top, bool zlive, f2 (&pn)[3]) {
        f2 gv = sub2(udown, uo), gh = sub2(uright, uo);
        if constexpr (!decltype(XYI)::value) {
            gv = i_lt ? gv : z2;
            gh = sel2(true, jlt_b, gh, z2);
        }
        f2 gz;
        if constexpr (decltype(ZI)::value) gz = sub2(uz, uo);
        else gz = top ? sub2(uz, uo) : z2;
        const f2 ph = fma2(gv, eta2, r[0]);
        const f2 qh = fma2(gh, eta2, r[1]);
        const f2 wh = fma2(gz, eta2, r[2]);
        const f2 inv = inv_norm2(fma2(wh, wh, fma2(qh, qh, mul2(ph, ph))));  // pinned order
        pn[0] = mul2(ph, inv);
        pn[1] = mul2(qh, inv);
        pn[2] = mul2(wh, inv);
        if constexpr (!(decltype(XYI)::value && decltype(ZI)::value)) {
            const bool live = zlive && inimg;
            pn[0] = live ? pn[0] : z2;
            pn[1] = live ? pn[1] : z2;
            pn[2] = live ? pn[2] : z2;
        }
    };

    int stg = 0;         // stage of plane s + 1
    uint32_t phase = 0;  // bit k: parity of stage k's next completion
    // One plane step; the two-deep registers are passed by role (prev / cur),
    // the parity-indexed delays (P_{k+1}, v) by their slot of this parity.
    auto step = [&](auto XYI, auto ZI, int s, f2 (&r0_prev)[3], f2 (&r0_cur)[3],
                    f2 (&r1_prev)[3], f2 (&r1_in)[3], f2 (&r2_prev)[3], f2 (&r2_in)[3],
                    f2 (&pk_prev)[3], f2 (&pk_cur)[3], f2 (&pd)[3], f2& u0_prev, f2& u0_cur,
                    f2& u1_prev, f2& u1_cur, f2& u2_prev, f2& u2_cur, f2& v_m1, f2& v_m3) {
        const int par = s & 1;
        mbar_wait((uint32_t)__cvta_generic_to_shared(&mbar[stg]), (phase >> stg) & 1u);
        phase ^= 1u << stg;
        const float* sp = fsm + stg * T::STAGE + own;
        const f2 v1 = ldx2(sp + 6 * T::PL);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            pk_cur[c] = ldx2(sp + c * T::PL);
            r0_cur[c] = fma2(sub2(pk_cur[c], ldx2(sp + (3 + c) * T::PL)), br2, pk_cur[c]);  // R_k(s + 1)
        }
        float* xr = XR + par * 6 * XPL;
        st2s(xr + 2 * tid, r0_cur[0]);
        st2s(xr + XPL + 2 * tid, r0_cur[1]);
        st2s(xr + 2 * XPL + 2 * tid, r1_in[0]);
        st2s(xr + 3 * XPL + 2 * tid, r1_in[1]);
        st2s(xr + 4 * XPL + 2 * tid, r2_in[0]);
        st2s(xr + 5 * XPL + 2 * tid, r2_in[1]);
        __syncthreads();  // exchange planes of step s written; step s - 1 fully read
        // the stage of plane s (read at step s - 1) takes plane s + NS
        if (tid == 0 && s >= pfirst && s + T::NS <= plast)
            issue(s + T::NS, stg == 0 ? T::NS - 1 : stg - 1);
        stg = stg + 1 == T::NS ? 0 : stg + 1;
        const float* xu_prev = XU + (par ^ 1) * 3 * XPL;
        float* xu = XU + par * 3 * XPL;
        const int z = a.z0 + s;
        // ---- phase 0: u_k(s + 1), P_{k+1}(s)
        u0_cur = u_of(XYI, ZI, r0_cur, ldx2(xr + 2 * n_up),
                      pk(xr[XPL + 2 * n_left + 1], lo_of(r0_cur[1])), r0_prev[2], v1,
                      z + 1 < Zg - 1, z + 1 > 0);
        st2s(xu + 2 * tid, u0_cur);
        f2 p1[3];
        dual(XYI, ZI, r0_prev, u0_prev, ldx2(xu_prev + 2 * n_down),
             pk(hi_of(u0_prev), xu_prev[2 * n_right]), u0_cur, z < Zg - 1, z >= 0 && z < Zg, p1);
        // ---- phase 1: u_{k+1}(s - 1), P_{k+2}(s - 2)
        u1_cur = u_of(XYI, ZI, r1_in, ldx2(xr + 2 * XPL + 2 * n_up),
                      pk(xr[3 * XPL + 2 * n_left + 1], lo_of(r1_in[1])), r1_prev[2], v_m1,
                      z - 1 < Zg - 1, z - 1 > 0);
        st2s(xu + XPL + 2 * tid, u1_cur);
        f2 p2[3];
        dual(XYI, ZI, r1_prev, u1_prev, ldx2(xu_prev + XPL + 2 * n_down),
             pk(hi_of(u1_prev), xu_prev[XPL + 2 * n_right]), u1_cur, z - 2 < Zg - 1,
             z - 2 >= 0 && z - 2 < Zg, p2);
        // ---- phase 2: u_{k+2}(s - 3), P_{k+3}(s - 4)
        u2_cur = u_of(XYI, ZI, r2_in, ldx2(xr + 4 * XPL + 2 * n_up),
                      pk(xr[5 * XPL + 2 * n_left + 1], lo_of(r2_in[1])), r2_prev[2], v_m3,
                      z - 3 < Zg - 1, z - 3 > 0);
        st2s(xu + 2 * XPL + 2 * tid, u2_cur);
        f2 p3[3];
        dual(XYI, ZI, r2_prev, u2_prev, ldx2(xu_prev + 2 * XPL + 2 * n_down),
             pk(hi_of(u2_prev), xu_prev[2 * XPL + 2 * n_right]), u2_cur, z - 4 < Zg - 1,
             z - 4 >= 0 && z - 4 < Zg, p3);
        // ---- outputs of the run's own planes (exact core only)
        o2 += plane3;
        o3 += plane3;
        if (core && s - 2 >= zb && s - 2 < ze) {
            st2s(o2, p2[0]); st2s(o2 + HW, p2[1]); st2s(o2 + 2 * HW, p2[2]);
        }
        if (core && s - 4 >= zb && s - 4 < ze) {
            st2s(o3, p3[0]); st2s(o3 + HW, p3[1]); st2s(o3 + 2 * HW, p3[2]);
        }
        // R_{k+2}(s - 2) for phase 2 takes the slot of R_{k+2}(s - 4), R_{k+1}(s)
        // for phase 1 that of R_{k+1}(s - 2) (both consumed above); P_{k+1}(s)
        // enters the two-step delay; v(s + 1) and v(s - 1) shift in
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            r2_prev[c] = fma2(sub2(p2[c], pd[c]), bk12, p2[c]);
            r1_prev[c] = fma2(sub2(p1[c], pk_prev[c]), bk2, p1[c]);
            pd[c] = p1[c];
        }
        v_m3 = v_m1;
        v_m1 = v1;
    };
    // roles: even steps (A) and odd steps (B); steps whose planes s - 4 .. s + 1
    // are all inside [1, Zg - 2] pass every z guard (ZI)
    auto march = [&](auto XYI) {
        const std::true_type zi{};
        const std::false_type zg{};
        int s = zb - 4;
        for (; s + 1 <= ze + 3; s += 2) {
            const int g0 = a.z0 + s;
            if (g0 - 4 >= 1 && g0 + 2 <= Zg - 2) {
                step(XYI, zi, s, r0a, r0b, r1a, r1b, r2a, r2b, pka, pkb, pda, u0a, u0b, u1a, u1b,
                     u2a, u2b, va, wa);
                step(XYI, zi, s + 1, r0b, r0a, r1b, r1a, r2b, r2a, pkb, pka, pdb, u0b, u0a, u1b,
                     u1a, u2b, u2a, vb, wb);
            } else {
                step(XYI, zg, s, r0a, r0b, r1a, r1b, r2a, r2b, pka, pkb, pda, u0a, u0b, u1a, u1b,
                     u2a, u2b, va, wa);
                step(XYI, zg, s + 1, r0b, r0a, r1b, r1a, r2b, r2a, pkb, pka, pdb, u0b, u0a, u1b,
                     u1a, u2b, u2a, vb, wb);
            }
        }
        if (s <= ze + 3)
            step(XYI, zg, s, r0a, r0b, r1a, r1b, r2a, r2b, pka, pkb, pda, u0a, u0b, u1a, u1b, u2a,
                 u2b, va, wa);
    };
    if (interior) march(std::true_type{});
    else march(std::false_type{});
    pdl_trigger<PDL_FGP3D>();
}

template <int BX2, int BY, int NS = 3>
static int fgp3d_col3_launch(Fgp3Args& a, int sm_count, cudaStream_t st)
{
    using T = Fgp3Col3<BX2, BY, NS>;
    const size_t smem = (size_t)T::SMEM_FLOATS * 4;
    {
        const int rc = ensure_smem((const void*)fgp3d_col3_kernel<BX2, BY, NS>, smem);
        if (rc) return rc;
    }
    int per_sm = 0;
    PT_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, fgp3d_col3_kernel<BX2, BY, NS>, T::NT, smem));
    Fgp3Maps m;
    memset(&m, 0, sizeof(m));
    const cuuint64_t W = a.W, H = a.H;
    const cuuint64_t d4[4] = {W, H, 3, (cuuint64_t)a.Zl + 2};
    const cuuint32_t b4[4] = {(cuuint32_t)T::BW, (cuuint32_t)BY, 3, 1};
    const cuuint64_t d3[3] = {W, H, (cuuint64_t)a.Zl};
    const cuuint32_t b3[3] = {(cuuint32_t)T::BW, (cuuint32_t)BY, 1};
    int rc = make_map(&m.R, a.R, 4, d4, b4);
    if (!rc) rc = make_map(&m.P, a.P, 4, d4, b4);
    if (!rc) rc = make_map(&m.V, a.v, 3, d3, b3);
    if (a.ghost) {  // z-slab: 3-plane ghosts of P_k, P_{k-1}, v a side
        const size_t HW = (size_t)a.W * a.H;
        const cuuint64_t g4[4] = {W, H, 3, 3};
        const cuuint64_t g3[3] = {W, H, 3};
        for (int side = 0; side < 2 && !rc; ++side) {
            const float* gb = a.ghost + (size_t)side * kGhostSide * HW;
            rc = make_map(&m.Rg[side], gb, 4, g4, b4);
            if (!rc) rc = make_map(&m.Pg[side], gb + kGhostPm * HW, 4, g4, b4);
            if (!rc) rc = make_map(&m.Vg[side], gb + kGhostV * HW, 3, g3, b3);
        }
    }
    if (rc) return rc;
    static const int zc_env = [] {
        const char* e = getenv("PT_FGP3_ZCHUNK");
        return e ? std::max(0, atoi(e)) : 0;
    }();
    const int tiles = ((a.W + T::CX - 1) / T::CX) * ((a.H + T::CY - 1) / T::CY);
    // z-runs: each re-marches 8 planes; as few runs as fill whole waves
    int zc = zc_env;
    if (!zc) {
        const int slots = sm_count * std::max(1, per_sm);
        int best_cost = INT32_MAX;
        zc = a.Zl;
        for (int c = 1; c <= std::max(1, a.Zl / 8); ++c) {
            const int run = (a.Zl + c - 1) / c;
            const int waves = (tiles * c + slots - 1) / slots;
            const int cost = waves * (run + 8);
            if (cost < best_cost) { best_cost = cost; zc = run; }
        }
    }
    a.zchunk = zc;
    const dim3 grid((a.W + T::CX - 1) / T::CX, (a.H + T::CY - 1) / T::CY,
                    (a.Zl + a.zchunk - 1) / a.zchunk);
    PT_CHECK_CUDA(launch_pdl(fgp3d_col3_kernel<BX2, BY, NS>, grid, dim3(T::NT), smem, st, a, m));
    PT_CHECK_LAUNCH();
    return PT_OK;
}

int fgp3d_run(const Fgp3Slab* sl, int G, int H, int W, int Zg, double lam, int inner,
              int nonneg, float pog, int64_t iteration, int64_t* bad_iter, const ZHalo* halo,
              int sm_count, cudaStream_t st)
{
    // TMA needs 16-byte row pitch; 64 x 8 tiles, 3-stage ring
    const bool tma = (W % 4) == 0 && tma_available();
    std::vector<double> betas(inner);
    double t = 1.0;
    for (int k = 0; k < inner; ++k) {
        const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        betas[k] = (t - 1.0) / tn;
        t = tn;
    }
    const size_t plane3 = 3 * (size_t)H * W;
    for (int g = 0; g < G; ++g) {
        const int Zl = sl[g].Zl;
        const size_t n = (size_t)Zl * H * W;
        const int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)sm_count * 16);
        fgp3d_pack_kernel<<<blocks, 256, 0, st>>>(sl[g].p, sl[g].q, sl[g].w,
                                                  fgp3d_set(sl[g].work, 0, Zl, H, W),
                                                  fgp3d_set(sl[g].work, 1, Zl, H, W), Zl, H, W);
        PT_CHECK_LAUNCH();
        // ghost planes on the global boundary stay zero (never exchanged)
        for (int k = 0; k < 4; ++k) {
            float* set = fgp3d_set(sl[g].work, k, Zl, H, W);
            if (sl[g].z0 == 0) PT_CHECK_CUDA(cudaMemsetAsync(set, 0, plane3 * 4, st));
            if (sl[g].z0 + Zl == Zg)
                PT_CHECK_CUDA(cudaMemsetAsync(set + (size_t)(Zl + 1) * plane3, 0, plane3 * 4, st));
        }
    }
    // One slab holding the whole volume: three iterations per pass (sets 0/1
    // and 2/3 alternate as {P_{k-1}, P_k} -> {P_{k+2}, P_{k+3}}; the first pass
    // reads set 0 twice, P_{-1} = P_0 with beta_r = 0), the remainder by a
    // two-iteration pass or the one-iteration kernel.  PT_FGP3_PAIR selects the
    // two-iteration kernel: 6 (default) the register-column kernel with
    // 32 x 16-point tiles; 5 / 7 / 8 other column tiles; 0 none (one iteration
    // per pass, no three-iteration passes either); PT_FGP3_TRIPLE=0 keeps two
    // iterations per pass.  256^3 FGP-100: 8.0 ms (three), 9.2 ms (two),
    // 14.0 ms (one); the windowed pair kernel of round 1: 11.7 ms.
    static const int pair_env = [] {
        const char* e = getenv("PT_FGP3_PAIR");
        return (e && *e) ? atoi(e) : 6;
    }();
    if (G == 1 && (!halo || halo->world <= 1) && tma && pair_env && inner >= 2 &&
        sl[0].z0 == 0 && sl[0].Zl == Zg) {
        const int Zl = sl[0].Zl;
        int rc = PT_OK;
        int sp = 0, sk = 0;  // sets of P_{k-1}, P_k
        int kk = 0;
        // three iterations per pass (PT_FGP3_TRIPLE=0: two), then a two-
        // iteration pass or a single iteration for the remainder
        static const bool triple = [] {
            const char* e = getenv("PT_FGP3_TRIPLE");
            return !(e && e[0] == '0');
        }();
        for (; triple && pair_env == 6 && kk + 3 <= inner; kk += 3) {
            const int o1 = (sk == 2 || sk == 3) ? 0 : 2;  // the pair not being read
            Fgp3Args a;
            a.Zl = Zl; a.H = H; a.W = W; a.z0 = 0; a.Zg = Zg;
            a.v = sl[0].v;
            a.vtop = nullptr;
            a.P = fgp3d_set(sl[0].work, sp, Zl, H, W);
            a.R = fgp3d_set(sl[0].work, sk, Zl, H, W);
            a.Pn = fgp3d_set(sl[0].work, o1, Zl, H, W);      // P_{k+2}
            a.Rn = fgp3d_set(sl[0].work, o1 + 1, Zl, H, W);  // P_{k+3}
            a.lam = (float)lam;
            a.eta = (float)(1.0 / (12.0 * lam));
            a.beta = (float)betas[kk];
            a.beta1 = (float)betas[kk + 1];
            a.beta_r = kk == 0 ? 0.f : (float)betas[kk - 1];
            a.nonneg = nonneg;
            // 32 x 32-point tiles, 3-stage ring: 256^3 FGP-100 8.0 ms (40 x 24 / 48 x 20 /
            // 32 x 24 points: 8.3 / 8.7 / 9.6 ms; a 4-stage ring 8.0 ms)
            rc = fgp3d_col3_launch<16, 32, 3>(a, sm_count, st);
            if (rc) return rc;
            sp = o1;
            sk = o1 + 1;
        }
        for (; kk + 2 <= inner; kk += 2) {
            const int o1 = (sk == 2 || sk == 3) ? 0 : 2;  // the pair not being read
            Fgp3Args a;
            a.Zl = Zl; a.H = H; a.W = W; a.z0 = 0; a.Zg = Zg;
            a.v = sl[0].v;
            a.vtop = nullptr;
            a.P = fgp3d_set(sl[0].work, sp, Zl, H, W);
            a.R = fgp3d_set(sl[0].work, sk, Zl, H, W);
            a.Pn = fgp3d_set(sl[0].work, o1, Zl, H, W);
            a.Rn = fgp3d_set(sl[0].work, o1 + 1, Zl, H, W);
            a.lam = (float)lam;
            a.eta = (float)(1.0 / (12.0 * lam));
            a.beta = (float)betas[kk];
            a.beta_r = kk == 0 ? 0.f : (float)betas[kk - 1];
            a.nonneg = nonneg;
            rc = pair_env == 5 ? fgp3d_col_launch<16, 16, 2>(a, sm_count, st)
               : pair_env == 7 ? fgp3d_col_launch<32, 16, 1>(a, sm_count, st)
               : pair_env == 8 ? fgp3d_col_launch<16, 24, 2>(a, sm_count, st)
                               : fgp3d_col_launch<16, 16, 3>(a, sm_count, st);
            if (rc) return rc;
            sp = o1;
            sk = o1 + 1;
        }
        if (kk < inner) {  // odd count: one more single iteration into a free set
            const int o = (sk == 2 || sk == 3) ? 0 : 2;
            Fgp3Args a;
            a.Zl = Zl; a.H = H; a.W = W; a.z0 = 0; a.Zg = Zg;
            a.v = sl[0].v;
            a.vtop = fgp3d_vtop(sl[0].work, Zl, H, W);
            a.P = fgp3d_set(sl[0].work, sp, Zl, H, W);
            a.R = fgp3d_set(sl[0].work, sk, Zl, H, W);
            a.Pn = fgp3d_set(sl[0].work, o, Zl, H, W);
            a.Rn = nullptr;
            a.lam = (float)lam;
            a.eta = (float)(1.0 / (12.0 * lam));
            a.beta = (float)betas[kk];
            a.beta_r = kk == 0 ? 0.f : (float)betas[kk - 1];
            a.nonneg = nonneg;
            rc = fgp3d_launch<64, 8, 3, true>(a, sm_count, st);
            if (rc) return rc;
            sk = o;
        }
        Fgp3Args a;
        a.Zl = Zl; a.H = H; a.W = W; a.z0 = 0; a.Zg = Zg;
        a.v = sl[0].v;
        a.P = fgp3d_set(sl[0].work, sk, Zl, H, W);
        a.lam = (float)lam;
        a.nonneg = nonneg;
        const size_t n = (size_t)Zl * H * W;
        const int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)sm_count * 16);
        PT_CHECK_CUDA(launch_pdl(fgp3d_final_kernel, dim3(blocks), dim3(256), 0, st, a, sl[0].p,
                                 sl[0].q, sl[0].w, sl[0].x_out, sl[0].xhat, sl[0].h, pog,
                                 (long long)iteration, (long long*)bad_iter));
        PT_CHECK_LAUNCH();
        return PT_OK;
    }
    // z-slabs (several local slabs and / or ranks) keep two iterations per HBM
    // pass: before each pass every slab receives the two boundary planes of
    // P_k and P_{k-1} of its neighbours (and of v, once per call) into its
    // 2-plane ghost buffers, which the column pass reads for planes -2, -1 and
    // Zl, Zl + 1 -- one exchange of 2-plane halos per two iterations instead of
    // one per iteration.  Every slab must hold >= 2 planes (decided from the
    // global plane count so that all ranks agree).
    const int ranks = (halo && halo->world > 1) ? halo->world : 1;
    bool col_slabs = tma && pair_env && inner >= 2 && Zg / (ranks * G) >= 2;
    for (int g = 0; g < G; ++g) col_slabs = col_slabs && sl[g].Zl >= 2;
    if (col_slabs) {
        int rc = PT_OK;
        for (int g = 0; g < G; ++g) {  // the volume's own boundary: zero ghosts
            if (sl[g].z0 == 0)
                PT_CHECK_CUDA(cudaMemsetAsync(fgp3d_ghost(sl[g].work, 0, sl[g].Zl, H, W), 0,
                                              kGhostSide * (size_t)H * W * 4, st));
            if (sl[g].z0 + sl[g].Zl == Zg)
                PT_CHECK_CUDA(cudaMemsetAsync(fgp3d_ghost(sl[g].work, 1, sl[g].Zl, H, W), 0,
                                              kGhostSide * (size_t)H * W * 4, st));
        }
        int sp = 0, sk = 0;  // sets of P_{k-1}, P_k (P_{-1} = P_0 with beta_r = 0)
        int kk = 0;
        // three iterations per pass with 3-plane ghosts when every slab holds
        // >= 3 planes (decided from the global plane count: all ranks agree)
        static const bool triple = [] {
            const char* e = getenv("PT_FGP3_TRIPLE");
            return !(e && e[0] == '0');
        }();
        bool tri = triple && pair_env == 6 && Zg / (ranks * G) >= 3;
        for (int g = 0; g < G; ++g) tri = tri && sl[g].Zl >= 3;
        for (; tri && kk + 3 <= inner; kk += 3) {
            rc = fgp3d_ghost_exchange(sl, G, H, W, sk, sp, kk == 0, halo, st, 3);
            if (rc) return rc;
            const int o1 = (sk == 2 || sk == 3) ? 0 : 2;
            for (int g = 0; g < G; ++g) {
                const int Zl = sl[g].Zl;
                Fgp3Args a;
                a.Zl = Zl; a.H = H; a.W = W; a.z0 = sl[g].z0; a.Zg = Zg;
                a.v = sl[g].v;
                a.vtop = nullptr;
                a.P = fgp3d_set(sl[g].work, sp, Zl, H, W);
                a.R = fgp3d_set(sl[g].work, sk, Zl, H, W);
                a.Pn = fgp3d_set(sl[g].work, o1, Zl, H, W);      // P_{k+2}
                a.Rn = fgp3d_set(sl[g].work, o1 + 1, Zl, H, W);  // P_{k+3}
                a.lam = (float)lam;
                a.eta = (float)(1.0 / (12.0 * lam));
                a.beta = (float)betas[kk];
                a.beta1 = (float)betas[kk + 1];
                a.beta_r = kk == 0 ? 0.f : (float)betas[kk - 1];
                a.nonneg = nonneg;
                a.ghost = fgp3d_ghost(sl[g].work, 0, Zl, H, W);
                rc = fgp3d_col3_launch<16, 32, 3>(a, sm_count, st);
                if (rc) return rc;
            }
            sp = o1;
            sk = o1 + 1;
        }
        // two iterations per pass (the remainder, or slabs of 2 planes); the
        // lower ghost slots of v hold planes -2, -1 only after a 2-plane exchange
        const int k2 = kk;
        for (; kk + 2 <= inner; kk += 2) {
            rc = fgp3d_ghost_exchange(sl, G, H, W, sk, sp, kk == k2, halo, st);
            if (rc) return rc;
            const int o1 = (sk == 2 || sk == 3) ? 0 : 2;
            for (int g = 0; g < G; ++g) {
                const int Zl = sl[g].Zl;
                Fgp3Args a;
                a.Zl = Zl; a.H = H; a.W = W; a.z0 = sl[g].z0; a.Zg = Zg;
                a.v = sl[g].v;
                a.vtop = nullptr;
                a.P = fgp3d_set(sl[g].work, sp, Zl, H, W);
                a.R = fgp3d_set(sl[g].work, sk, Zl, H, W);
                a.Pn = fgp3d_set(sl[g].work, o1, Zl, H, W);
                a.Rn = fgp3d_set(sl[g].work, o1 + 1, Zl, H, W);
                a.lam = (float)lam;
                a.eta = (float)(1.0 / (12.0 * lam));
                a.beta = (float)betas[kk];
                a.beta_r = kk == 0 ? 0.f : (float)betas[kk - 1];
                a.nonneg = nonneg;
                a.ghost = fgp3d_ghost(sl[g].work, 0, Zl, H, W);
                rc = fgp3d_col_launch<16, 16, 3>(a, sm_count, st);
                if (rc) return rc;
            }
            sp = o1;
            sk = o1 + 1;
        }
        if (kk < inner) {  // odd count: one more single iteration (one-plane set ghosts)
            rc = fgp3d_exchange(sl, G, H, W, sk, true, halo, st);
            if (!rc) rc = fgp3d_exchange(sl, G, H, W, sp, false, halo, st);
            if (rc) return rc;
            const int o = (sk == 2 || sk == 3) ? 0 : 2;
            for (int g = 0; g < G; ++g) {
                const int Zl = sl[g].Zl;
                Fgp3Args a;
                a.Zl = Zl; a.H = H; a.W = W; a.z0 = sl[g].z0; a.Zg = Zg;
                a.v = sl[g].v;
                a.vtop = fgp3d_vtop(sl[g].work, Zl, H, W);
                a.P = fgp3d_set(sl[g].work, sp, Zl, H, W);
                a.R = fgp3d_set(sl[g].work, sk, Zl, H, W);
                a.Pn = fgp3d_set(sl[g].work, o, Zl, H, W);
                a.Rn = nullptr;
                a.lam = (float)lam;
                a.eta = (float)(1.0 / (12.0 * lam));
                a.beta = (float)betas[kk];
                a.beta_r = kk == 0 ? 0.f : (float)betas[kk - 1];
                a.nonneg = nonneg;
                rc = fgp3d_launch<64, 8, 3, true>(a, sm_count, st);
                if (rc) return rc;
            }
            sk = o;
        }
        rc = fgp3d_exchange(sl, G, H, W, sk, false, halo, st);  // P ghost below for D^T
        if (rc) return rc;
        for (int g = 0; g < G; ++g) {
            const int Zl = sl[g].Zl;
            Fgp3Args a;
            a.Zl = Zl; a.H = H; a.W = W; a.z0 = sl[g].z0; a.Zg = Zg;
            a.v = sl[g].v;
            a.P = fgp3d_set(sl[g].work, sk, Zl, H, W);
            a.lam = (float)lam;
            a.nonneg = nonneg;
            const size_t n = (size_t)Zl * H * W;
            const int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)sm_count * 16);
            PT_CHECK_CUDA(launch_pdl(fgp3d_final_kernel, dim3(blocks), dim3(256), 0, st, a,
                                     sl[g].p, sl[g].q, sl[g].w, sl[g].x_out, sl[g].xhat, sl[g].h,
                                     pog, (long long)iteration, (long long*)bad_iter));
            PT_CHECK_LAUNCH();
        }
        return PT_OK;
    }
    // one iteration per pass: sets 0, 1, 2 rotate P_{k-1}, P_k -> P_{k+1}
    int rc = fgp3d_exchange(sl, G, H, W, 0, true, halo, st);
    if (rc) return rc;
    for (int kk = 0; kk < inner; ++kk) {
        const int set_r = kk % 3;                      // P_k (windows)
        const int set_p = kk == 0 ? 0 : (kk + 2) % 3;  // P_{k-1}
        const int set_pn = (kk + 1) % 3;
        for (int g = 0; g < G; ++g) {
            const int Zl = sl[g].Zl;
            Fgp3Args a;
            a.Zl = Zl; a.H = H; a.W = W; a.z0 = sl[g].z0; a.Zg = Zg;
            a.v = sl[g].v;
            a.vtop = fgp3d_vtop(sl[g].work, Zl, H, W);
            a.P = fgp3d_set(sl[g].work, set_p, Zl, H, W);
            a.R = fgp3d_set(sl[g].work, set_r, Zl, H, W);
            a.Pn = fgp3d_set(sl[g].work, set_pn, Zl, H, W);
            a.Rn = nullptr;
            a.lam = (float)lam;
            a.eta = (float)(1.0 / (12.0 * lam));
            a.beta = (float)betas[kk];
            a.beta_r = kk == 0 ? 0.f : (float)betas[kk - 1];
            a.nonneg = nonneg;
            rc = tma ? fgp3d_launch<64, 8, 3, true>(a, sm_count, st)
                     : fgp3d_launch<32, 8, 3, false>(a, sm_count, st);
            if (rc) return rc;
        }
        rc = fgp3d_exchange(sl, G, H, W, set_pn, false, halo, st);
        if (rc) return rc;
    }
    const int fin = inner % 3;
    for (int g = 0; g < G; ++g) {
        const int Zl = sl[g].Zl;
        Fgp3Args a;
        a.Zl = Zl; a.H = H; a.W = W; a.z0 = sl[g].z0; a.Zg = Zg;
        a.v = sl[g].v;
        a.P = fgp3d_set(sl[g].work, fin, Zl, H, W);
        a.lam = (float)lam;
        a.nonneg = nonneg;
        const size_t n = (size_t)Zl * H * W;
        const int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)sm_count * 16);
        PT_CHECK_CUDA(launch_pdl(fgp3d_final_kernel, dim3(blocks), dim3(256), 0, st, a, sl[g].p,
                                 sl[g].q, sl[g].w, sl[g].x_out, sl[g].xhat, sl[g].h, pog,
                                 (long long)iteration, (long long*)bad_iter));
        PT_CHECK_LAUNCH();
    }
    return PT_OK;
}

int launch_tv_prox(pt_plan* plan, const float* v, double lam, int inner, int nonneg, float* p,
                   float* q, float* w, float* x_out, const float* xhat, float* h,
                   float p_over_gamma, int64_t iteration, int64_t* bad_iter, float* work,
                   cudaStream_t st)
{
    if (inner < 1) {
        set_error("inner_iterations must be >= 1");
        return PT_EINVAL;
    }
    if (plan->Z > 1) {
        Fgp3Slab sl;
        sl.Zl = plan->Z; sl.z0 = 0;
        sl.v = v; sl.p = p; sl.q = q; sl.w = w;
        sl.x_out = x_out; sl.xhat = xhat; sl.h = h; sl.work = work;
        return fgp3d_run(&sl, 1, plan->H, plan->W, plan->Z, lam, inner, nonneg, p_over_gamma,
                         iteration, bad_iter, nullptr, plan->sm_count, st);
    }
    if (fgp2d_big(plan->H, plan->W))
        return run_fgp2d<64, 64, 8>(plan, v, lam, inner, nonneg, p, q, x_out, xhat, h,
                                    p_over_gamma, iteration, bad_iter, work, st,
                                    fgp2d_tmax(plan->H, plan->W));
    static const int t_small = [] {
        const char* e = getenv("PT_FGP_T_SMALL");
        return e ? std::max(1, std::min(kFgpMaxT, atoi(e))) : 10;
    }();
    return run_fgp2d<32, 32, 8>(plan, v, lam, inner, nonneg, p, q, x_out, xhat, h,
                                p_over_gamma, iteration, bad_iter, work, st, t_small);
}

}  // namespace pt
