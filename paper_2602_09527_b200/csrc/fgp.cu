// FGP (Beck-Teboulle fast gradient projection on the dual) TV prox for
// sm_100a, temporally blocked: one launch runs T inner iterations on a
// (RH x RW) region held on chip, of which the central (RH-2T-2) x (RW-2T-2)
// points are exact after T iterations (each iteration's stencil reaches one
// point further, pkg/src/proxtomo/regularizers.py:62-76); only those are
// written back.  So a prox call with n inner iterations costs ceil(n/T)
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
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "pt_internal.cuh"
#include "pt_simd.cuh"

namespace pt {

struct FgpArgs {
    int H, W;
    const float* v;
    const float *p_in, *q_in, *r_in, *s_in;  // r_in == nullptr: r = p, s = q (call start)
    float *p_out, *q_out, *r_out, *s_out;
    float lam, eta;
    float beta[8];
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

// One FGP inner iteration on the register strips.  EDGE = the region touches
// the image border (masks needed); interior regions skip every boundary test.
template <int RW, int RH, int STRIP, bool EDGE>
__device__ __forceinline__ void fgp2d_iteration(
    float (&v)[STRIP], float (&p)[STRIP], float (&q)[STRIP], float (&r)[STRIP],
    float (&s)[STRIP], float (&u)[STRIP], float (*S_s)[RW + 1], float (*S_u)[RW + 1],
    float (*S_r)[RW], float (*S_ut)[RW], int tx, int ty, int i0, int H, bool not_last_col,
    unsigned in_mask, float lam, float eta, float beta, int nonneg)
{
    constexpr int NS = RH / STRIP;
    const int row0 = ty * STRIP;
#pragma unroll
    for (int k = 0; k < STRIP; ++k) S_s[row0 + k][tx] = s[k];
    S_r[ty][tx] = r[STRIP - 1];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < STRIP; ++k) {
        const float r_up = k ? r[k - 1] : (ty ? S_r[ty - 1][tx] : 0.f);
        const float s_left = tx ? S_s[row0 + k][tx - 1] : 0.f;
        // _diff_adjoint (regularizers.py:70-76), numpy statement order
        float o;
        if (EDGE) {
            const int gi = i0 + row0 + k;
            o = (gi < H - 1) ? -r[k] : 0.f;
            o += r_up;
            o = not_last_col ? o - s[k] : o;
        } else {
            o = -r[k];
            o += r_up;
            o = o - s[k];
        }
        o += s_left;
        float uu = v[k] - lam * o;
        if (nonneg) uu = (uu < 0.f) ? 0.f : uu;
        if (EDGE) uu = ((in_mask >> k) & 1u) ? uu : 0.f;
        u[k] = uu;
        S_u[row0 + k][tx] = uu;
    }
    S_ut[ty][tx] = u[0];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < STRIP; ++k) {
        const float u_down = (k < STRIP - 1) ? u[k + 1] : (ty < NS - 1 ? S_ut[ty + 1][tx] : 0.f);
        const float u_right = (tx < RW - 1) ? S_u[row0 + k][tx + 1] : 0.f;
        float gv = u_down - u[k], gh = u_right - u[k];
        if (EDGE) {
            const int gi = i0 + row0 + k;
            gv = (gi < H - 1) ? gv : 0.f;
            gh = not_last_col ? gh : 0.f;
        }
        const float ph = r[k] + eta * gv;
        const float qh = s[k] + eta * gh;
        const float n2 = ph * ph + qh * qh;
        const float inv = (n2 > 1.f) ? rsqrtf(n2) : 1.f;
        const float pn = ph * inv, qn = qh * inv;
        if (!EDGE || ((in_mask >> k) & 1u)) {
            r[k] = pn + beta * (pn - p[k]);
            s[k] = qn + beta * (qn - q[k]);
            p[k] = pn;
            q[k] = qn;
        }
    }
}

// Interior iteration with packed f32x2 arithmetic.  A thread's strip rows are
// held as pairs (j, j + H2), H2 = STRIP/2, so the up-neighbour of pair j is
// pair j-1 and the down-neighbour of pair j is pair j+1 (one repack at the
// strip ends): the stencil needs no lane shuffling.  The left/right exchange
// planes store the pairs as float2 (one 64-bit LDS/STS per pair, operands land
// in aligned register pairs).
__device__ __forceinline__ float rsqrt_ftz(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
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

template <int RW, int RH, int STRIP>
__device__ __forceinline__ void fgp2d_iteration_packed(
    f2 (&V)[STRIP / 2], f2 (&Pp)[STRIP / 2], f2 (&Q)[STRIP / 2], f2 (&R)[STRIP / 2],
    f2 (&S)[STRIP / 2], f2 (&U)[STRIP / 2], float2 (*S_s2)[RW + 1], float2 (*S_u2)[RW + 1],
    float (*S_r)[RW], float (*S_ut)[RW], int tx, int ty, float lam, float eta, float beta,
    int nonneg)
{
    constexpr int NS = RH / STRIP;
    constexpr int H2 = STRIP / 2;
    const int prow0 = ty * H2;
    const f2 nlam2 = pk(-lam, -lam), eta2 = pk(eta, eta), beta2 = pk(beta, beta);
    const f2 zero2 = pk(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < H2; ++j) st2(&S_s2[prow0 + j][tx], S[j]);
    S_r[ty][tx] = hi_of(R[H2 - 1]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < H2; ++j) {
        const f2 r_up = j ? R[j - 1] : pk(ty ? S_r[ty - 1][tx] : 0.f, lo_of(R[H2 - 1]));
        const f2 s_left = tx ? ld2(&S_s2[prow0 + j][tx - 1]) : zero2;
        // _diff_adjoint (regularizers.py:70-76): ((-r + r_up) - s) + s_left
        const f2 o = add2(sub2(sub2(r_up, R[j]), S[j]), s_left);
        f2 u = fma2(nlam2, o, V[j]);
        if (nonneg) {
            float ua, ub;
            upk(u, ua, ub);
            u = pk((ua < 0.f) ? 0.f : ua, (ub < 0.f) ? 0.f : ub);  // NaN propagates
        }
        U[j] = u;
        st2(&S_u2[prow0 + j][tx], u);
    }
    S_ut[ty][tx] = lo_of(U[0]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < H2; ++j) {
        // rows (j+1, j+1+H2); for the last pair: (pair 0 hi, next strip's first row)
        const f2 u_down = (j < H2 - 1) ? U[j + 1]
                                       : pk(hi_of(U[0]), ty < NS - 1 ? S_ut[ty + 1][tx] : 0.f);
        const f2 u_right = (tx < RW - 1) ? ld2(&S_u2[prow0 + j][tx + 1]) : zero2;
        const f2 gv = sub2(u_down, U[j]);
        const f2 gh = sub2(u_right, U[j]);
        const f2 ph = fma2(eta2, gv, R[j]);
        const f2 qh = fma2(eta2, gh, S[j]);
        const f2 n2 = fma2(ph, ph, mul2(qh, qh));
        float na, nb;
        upk(n2, na, nb);
        // max(1, |.|): the projection only rescales when |.| > 1 (no denormals there)
        const f2 inv = pk((na > 1.f) ? rsqrt_ftz(na) : 1.f, (nb > 1.f) ? rsqrt_ftz(nb) : 1.f);
        const f2 pn = mul2(ph, inv), qn = mul2(qh, inv);
        R[j] = fma2(beta2, sub2(pn, Pp[j]), pn);
        S[j] = fma2(beta2, sub2(qn, Q[j]), qn);
        Pp[j] = pn;
        Q[j] = qn;
    }
}

template <int RW, int RH, int STRIP>
__global__ void __launch_bounds__(RW*(RH / STRIP), 2) fgp2d_kernel(FgpArgs P)
{
    constexpr int H2 = STRIP / 2;
    // the scalar (edge / epilogue) and the pair (interior) exchange planes
    // share one buffer: a CTA uses one layout at a time
    __shared__ __align__(16) float S_buf[2 * RH * (RW + 1)];
    float (*S_s)[RW + 1] = reinterpret_cast<float (*)[RW + 1]>(S_buf);
    float (*S_u)[RW + 1] = reinterpret_cast<float (*)[RW + 1]>(S_buf + RH * (RW + 1));
    float2 (*S_s2)[RW + 1] = reinterpret_cast<float2 (*)[RW + 1]>(S_buf);
    float2 (*S_u2)[RW + 1] = reinterpret_cast<float2 (*)[RW + 1]>(S_buf + RH * (RW + 1));
    __shared__ float S_r[RH / STRIP][RW];
    __shared__ float S_ut[RH / STRIP][RW];

    const int tid = threadIdx.x;
    const int tx = tid % RW;
    const int ty = tid / RW;
    const int IW = RW - 2 * P.halo, IH = RH - 2 * P.halo;
    const int j0 = blockIdx.x * IW - P.halo;
    const int i0 = blockIdx.y * IH - P.halo;
    const int gj = j0 + tx;
    const int row0 = ty * STRIP;
    const bool col_in = (gj >= 0 && gj < P.W);
    const bool not_last_col = (gj < P.W - 1);
    // the whole region, and one point beyond it, strictly inside the image
    const bool edge = !(i0 >= 0 && j0 >= 0 && i0 + RH < P.H && j0 + RW < P.W);

    // packed state: pair j = strip rows (j, j + H2)
    f2 V[H2], Pp[H2], Q[H2], R[H2], S[H2], U[H2];
    unsigned in_mask = 0;
#pragma unroll
    for (int j = 0; j < H2; ++j) {
        float vv[2], pv[2], qv[2], rv[2], sv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = j + h * H2;
            const int gi = i0 + row0 + k;
            const bool in = col_in && gi >= 0 && gi < P.H;
            if (in) in_mask |= 1u << k;
            const size_t o = in ? (size_t)gi * P.W + gj : 0;
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
    for (int it = 0; it < P.n_iter; ++it) {
        if (!edge) {
            fgp2d_iteration_packed<RW, RH, STRIP>(V, Pp, Q, R, S, U, S_s2, S_u2, S_r, S_ut, tx, ty,
                                                  P.lam, P.eta, P.beta[it], P.nonneg);
        } else {
            float v[STRIP], p[STRIP], q[STRIP], r[STRIP], s[STRIP], u[STRIP];
#pragma unroll
            for (int j = 0; j < H2; ++j) {
                upk(V[j], v[j], v[j + H2]);
                upk(Pp[j], p[j], p[j + H2]);
                upk(Q[j], q[j], q[j + H2]);
                upk(R[j], r[j], r[j + H2]);
                upk(S[j], s[j], s[j + H2]);
                upk(U[j], u[j], u[j + H2]);
            }
            fgp2d_iteration<RW, RH, STRIP, true>(v, p, q, r, s, u, S_s, S_u, S_r, S_ut, tx, ty, i0,
                                                 P.H, not_last_col, in_mask, P.lam, P.eta,
                                                 P.beta[it], P.nonneg);
#pragma unroll
            for (int j = 0; j < H2; ++j) {
                Pp[j] = pk(p[j], p[j + H2]);
                Q[j] = pk(q[j], q[j + H2]);
                R[j] = pk(r[j], r[j + H2]);
                S[j] = pk(s[j], s[j + H2]);
                U[j] = pk(u[j], u[j + H2]);
            }
        }
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
    const bool col_inner = tx >= P.halo && tx < RW - P.halo;
    const float lam = P.lam;
    if (P.final_) {
        // x = max(v - lam D^T(p, q), 0), then the ProxSkip h update
        __syncthreads();
#pragma unroll
        for (int k = 0; k < STRIP; ++k) S_s[row0 + k][tx] = q[k];
        S_r[ty][tx] = p[STRIP - 1];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < STRIP; ++k) {
            const int li = row0 + k;
            const int gi = i0 + li;
            if (!col_inner || li < P.halo || li >= RH - P.halo || !((in_mask >> k) & 1u)) continue;
            const float p_up = k ? p[k - 1] : (ty ? S_r[ty - 1][tx] : 0.f);
            const float q_left = tx ? S_s[li][tx - 1] : 0.f;
            float o = (gi < P.H - 1) ? -p[k] : 0.f;
            o += p_up;
            o = not_last_col ? o - q[k] : o;
            o += q_left;
            float x = v[k] - lam * o;
            if (P.nonneg) x = (x < 0.f) ? 0.f : x;
            const size_t idx = (size_t)gi * P.W + gj;
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
            const int li = row0 + k;
            const int gi = i0 + li;
            if (!col_inner || li < P.halo || li >= RH - P.halo || !((in_mask >> k) & 1u)) continue;
            const size_t idx = (size_t)gi * P.W + gj;
            P.p_out[idx] = p[k];
            P.q_out[idx] = q[k];
            P.r_out[idx] = r[k];
            P.s_out[idx] = s[k];
        }
    }
}

int64_t fgp_workspace_floats(const pt_plan* plan)
{
    // two ping-pong sets of (p, q, r, s) [2D] or (p, q, w, r, s, t) [3D]
    const int64_t n = (int64_t)plan->Z * plan->H * plan->W;
    return plan->Z > 1 ? 12 * n : 8 * n;
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
        for (int k = 0; k < 8; ++k) a.beta[k] = (k < iters) ? (float)betas[done + k] : 0.f;
        a.n_iter = iters;
        a.halo = iters + 1;
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
        fgp2d_kernel<RW, RH, STRIP><<<grid, RW * (RH / STRIP), 0, st>>>(a);
        PT_CHECK_LAUNCH();
        if (!fin) {
            sp = D[0]; sq = D[1]; sr = D[2]; ss = D[3];
        }
        done += iters;
    }
    return PT_OK;
}

// ---------------------------------------------------------------------------
// 3D isotropic FGP on a (Z, H, W) volume (slice-stacked geometry, config 3).
// No reference code exists: the 2D algorithm with a
// third forward difference along z and dual step 1/(12 lam).  Two passes per
// inner iteration: u from the dual neighbours, then the pointwise dual update.
// ---------------------------------------------------------------------------
struct Fgp3Args {
    int Z, H, W;
    const float* v;
    const float *r, *s, *t;  // momentum duals (read in the u pass)
    float *pp, *qq, *ww;     // duals
    float *rr, *ss, *tt;     // momentum duals (written in the dual pass)
    float* u;
    float lam, eta, beta;
    int nonneg;
};

__device__ __forceinline__ float dt3(const float* a, const float* b, const float* c, int Z, int H,
                                     int W, int k, int i, int j, size_t o)
{
    const size_t plane = (size_t)H * W;
    float x = (i < H - 1) ? -a[o] : 0.f;
    if (i > 0) x += a[o - W];
    if (j < W - 1) x -= b[o];
    if (j > 0) x += b[o - 1];
    if (k < Z - 1) x -= c[o];
    if (k > 0) x += c[o - plane];
    return x;
}

__global__ void fgp3d_u_kernel(Fgp3Args P)
{
    const size_t n = (size_t)P.Z * P.H * P.W;
    for (size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
         o += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(o % P.W);
        const size_t t1 = o / P.W;
        const int i = (int)(t1 % P.H);
        const int k = (int)(t1 / P.H);
        float uu = P.v[o] - P.lam * dt3(P.r, P.s, P.t, P.Z, P.H, P.W, k, i, j, o);
        if (P.nonneg) uu = (uu < 0.f) ? 0.f : uu;
        P.u[o] = uu;
    }
}

__global__ void fgp3d_dual_kernel(Fgp3Args P)
{
    const size_t n = (size_t)P.Z * P.H * P.W;
    const size_t plane = (size_t)P.H * P.W;
    for (size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
         o += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(o % P.W);
        const size_t t1 = o / P.W;
        const int i = (int)(t1 % P.H);
        const int k = (int)(t1 / P.H);
        const float uo = P.u[o];
        const float gv = (i < P.H - 1) ? P.u[o + P.W] - uo : 0.f;
        const float gh = (j < P.W - 1) ? P.u[o + 1] - uo : 0.f;
        const float gz = (k < P.Z - 1) ? P.u[o + plane] - uo : 0.f;
        const float ph = P.rr[o] + P.eta * gv;
        const float qh = P.ss[o] + P.eta * gh;
        const float wh = P.tt[o] + P.eta * gz;
        const float n2 = ph * ph + qh * qh + wh * wh;
        const float inv = (n2 > 1.f) ? rsqrtf(n2) : 1.f;
        const float pn = ph * inv, qn = qh * inv, wn = wh * inv;
        P.rr[o] = pn + P.beta * (pn - P.pp[o]);
        P.ss[o] = qn + P.beta * (qn - P.qq[o]);
        P.tt[o] = wn + P.beta * (wn - P.ww[o]);
        P.pp[o] = pn;
        P.qq[o] = qn;
        P.ww[o] = wn;
    }
}

__global__ void fgp3d_final_kernel(Fgp3Args P, float* x_out, const float* xhat, float* h,
                                   float pog, long long iteration, long long* bad_iter)
{
    const size_t n = (size_t)P.Z * P.H * P.W;
    for (size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
         o += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(o % P.W);
        const size_t t1 = o / P.W;
        const int i = (int)(t1 % P.H);
        const int k = (int)(t1 / P.H);
        float x = P.v[o] - P.lam * dt3(P.pp, P.qq, P.ww, P.Z, P.H, P.W, k, i, j, o);
        if (P.nonneg) x = (x < 0.f) ? 0.f : x;
        x_out[o] = x;
        if (h) h[o] = h[o] + pog * (x - xhat[o]);
        if (!isfinite(x) && bad_iter) atomicMin(bad_iter, iteration);
    }
}

int launch_fgp3d(pt_plan* plan, const float* v, double lam, int inner, int nonneg, float* p,
                 float* q, float* w, float* x_out, const float* xhat, float* h, float pog,
                 int64_t iteration, int64_t* bad_iter, float* work, cudaStream_t st)
{
    const size_t n = (size_t)plan->Z * plan->H * plan->W;
    Fgp3Args a;
    a.Z = plan->Z; a.H = plan->H; a.W = plan->W;
    a.v = v;
    a.pp = p; a.qq = q; a.ww = w;
    a.rr = work; a.ss = work + n; a.tt = work + 2 * n;
    a.u = work + 3 * n;
    a.r = a.rr; a.s = a.ss; a.t = a.tt;
    a.lam = (float)lam;
    a.eta = (float)(1.0 / (12.0 * lam));
    a.nonneg = nonneg;
    PT_CHECK_CUDA(cudaMemcpyAsync(a.rr, p, n * 4, cudaMemcpyDeviceToDevice, st));
    PT_CHECK_CUDA(cudaMemcpyAsync(a.ss, q, n * 4, cudaMemcpyDeviceToDevice, st));
    PT_CHECK_CUDA(cudaMemcpyAsync(a.tt, w, n * 4, cudaMemcpyDeviceToDevice, st));
    const int blocks = (int)std::min<size_t>((n + 255) / 256, (size_t)plan->sm_count * 16);
    double t = 1.0;
    for (int kk = 0; kk < inner; ++kk) {
        const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        a.beta = (float)((t - 1.0) / tn);
        t = tn;
        fgp3d_u_kernel<<<blocks, 256, 0, st>>>(a);
        PT_CHECK_LAUNCH();
        fgp3d_dual_kernel<<<blocks, 256, 0, st>>>(a);
        PT_CHECK_LAUNCH();
    }
    fgp3d_final_kernel<<<blocks, 256, 0, st>>>(a, x_out, xhat, h, pog, (long long)iteration,
                                               (long long*)bad_iter);
    PT_CHECK_LAUNCH();
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
    if (plan->Z > 1)
        return launch_fgp3d(plan, v, lam, inner, nonneg, p, q, w, x_out, xhat, h, p_over_gamma,
                            iteration, bad_iter, work, st);
    if (std::min(plan->H, plan->W) >= 256)
    {
        static const int tmax = [] {
            const char* e = getenv("PT_FGP_T");
            return e ? std::max(1, std::min(8, atoi(e))) : 6;
        }();
        return run_fgp2d<64, 64, 8>(plan, v, lam, inner, nonneg, p, q, x_out, xhat, h,
                                    p_over_gamma, iteration, bad_iter, work, st, tmax);
    }
    return run_fgp2d<32, 32, 8>(plan, v, lam, inner, nonneg, p, q, x_out, xhat, h,
                                p_over_gamma, iteration, bad_iter, work, st, 3);
}

}  // namespace pt
