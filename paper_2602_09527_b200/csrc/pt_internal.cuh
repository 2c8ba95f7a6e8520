// Internal declarations shared by the sm_100a kernels and the C ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/proxtomo_b200.h"

namespace pt {

// Per-angle Joseph parameters, computed on the host in float64 from the
// reference expressions (pkg/src/proxtomo/projector.py:28-51):
//   pos(b, step) = a0 + b * sigma + step * m     (in lane units)
// branch 0: |cos| >= |sin|, one sample per image row, lanes = columns
//           sigma = ds/(h cos), m = -tan, a0 = -cB sigma + cH tan + cW
// branch 1: one sample per image column, lanes = rows
//           sigma = ds/(h sin), m = -cot, a0 = -cB sigma + cW cot + cH
// with cB = (B-1)/2, cH = (H-1)/2, cW = (W-1)/2; step_len = h/max(|cos|,|sin|).
struct AngleTab {
    double sigma, m, a0;
    double isig, im;  // 1/sigma, 1/m (0 when m == 0)
    // gather: crossing bin b_f(r, c) = gbr*r + gbc*c + gg, where pos(b_f) == lane
    double gbr, gbc, gg;
    float step_len;
    int branch;
};

void set_error(const char* fmt, ...);

#define PT_CHECK_CUDA(call)                                                          \
    do {                                                                             \
        cudaError_t e_ = (call);                                                     \
        if (e_ != cudaSuccess) {                                                     \
            ::pt::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,               \
                            cudaGetErrorString(e_));                                 \
            return PT_ECUDA;                                                         \
        }                                                                            \
    } while (0)

extern std::atomic<long long> g_launches;  // kernels launched by this library

#define PT_CHECK_LAUNCH()      \
    do {                       \
        ::pt::g_launches++;    \
        PT_CHECK_CUDA(cudaGetLastError()); \
    } while (0)

// Programmatic dependent launch (PDL).  The solver's kernels are launched
// with programmatic stream serialisation: a kernel may start while its
// predecessor drains, runs only predecessor-independent prologue work, then
// pdl_wait() (griddepcontrol.wait: the predecessor grid has completed and its
// writes are visible).  A kernel family releases its successor either at its
// end, after its last global write (the default), or right after its own wait
// (its bit set in PT_PDL_EARLY_MASK: the successor's CTAs become resident as
// this grid's last CTAs retire and block at their own wait).  Either way, when
// kernel N+1 is released some thread of kernel N has passed its wait, so
// kernels <= N-1 are complete -- N+1's prologue may read their outputs, never
// kernel N's (nor any buffer kernel N writes).  Measured per family
// (tools/ab/pdl_mask.sh, profiles/ANALYSIS_r02.md): only the one-launch small
// forward gains from the early release (config 0 +7.7%: its successor, the
// gather, stages its operands while the forward's single wave drains); an
// early release everywhere is slower (config 1 -17%: the successor's CTAs
// pile onto the SMs that drain first instead of spreading over all of them).
// Kernels launched without the attribute see both as no-ops.
#ifndef PT_PDL_EARLY_MASK
#define PT_PDL_EARLY_MASK 2  // PDL_FWD_SMALL
#endif
enum : int {
    PDL_FWD = 1, PDL_FWD_SMALL = 2, PDL_REDUCE = 4, PDL_GATHER = 8, PDL_FGP2D = 16,
    PDL_FGP3D = 32, PDL_MISC = 64
};
template <int F = PDL_MISC>
__device__ __forceinline__ void pdl_wait()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if constexpr ((PT_PDL_EARLY_MASK & F) != 0)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <int F = PDL_MISC>
__device__ __forceinline__ void pdl_trigger()
{
    if constexpr ((PT_PDL_EARLY_MASK & F) == 0)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();

// Raise a kernel's dynamic shared-memory limit to `bytes` on the current
// device (once per (kernel, device, size); thread-safe, multi-device safe).
int ensure_smem(const void* kernel, size_t bytes);

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace pt

struct pt_selection {
    int32_t n = 0;
    std::vector<int32_t> h_angle;       // geometry angle index per selection slot
    int32_t* d_angle = nullptr;         // [n]
    int32_t n_branch[2] = {0, 0};
    int32_t* d_branch_pos[2] = {nullptr, nullptr};  // selection slots per branch
    int64_t nnz = -1;
};

namespace pt {
// Gather pixel tiles (rows x columns), 256 threads each: 0 = 32 x 128 (16
// pixels per thread, large images), 1 = 32 x 64 (8), 2 = 16 x 64 (4, small
// images: enough CTAs).  The plan picks one and sizes its staged-bin slot per
// angle for that tile (capi.cu).
constexpr int kGatherTiles[4][2] = {{32, 128}, {32, 64}, {16, 64}, {8, 64}};
constexpr int kGatherNA = 32;  // angles per staged gather chunk

// Per-caller scratch for the forward band partials and reductions.  The plan
// owns one (used by the standalone C-ABI calls, which must therefore be
// stream-serialised per plan, like a cuFFT plan); every session owns its own.
// Optional per-kernel device timing (CUDA events around launches on the
// caller's stream), used by bench.py for the live roofline.
struct Profiler {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    struct Rec { int cat; size_t ev0; };
    std::vector<Rec> recs;
    // open scopes: index into recs, or -1 for a nested scope that does not
    // record (only the outermost scope records, except that the kernel
    // scopes inside a snapshot record as the PT_PROF_SNAP_* categories)
    std::vector<long> open;
    int outer = -1;  // category of the outermost open scope
    double ms[PT_PROF_N] = {0};
    long long calls[PT_PROF_N] = {0};
    cudaEvent_t ev();
    void begin(int cat, cudaStream_t st);  // pairs: begin, then end
    void end(cudaStream_t st);
    int collect();
    ~Profiler();
};
struct Workspace {
    float* partial = nullptr;
    size_t partial_floats = 0;
    double* red = nullptr;
    size_t red_doubles = 0;
    float* image = nullptr;  // image-sized temp (difference images)
    size_t image_floats = 0;
    Profiler* prof = nullptr;
};
struct ProfScope {
    Profiler* p;
    cudaStream_t st;
    ProfScope(Workspace* ws, int cat, cudaStream_t s) : p(ws && ws->prof && ws->prof->on ? ws->prof : nullptr), st(s)
    {
        if (p) p->begin(cat, st);
    }
    ~ProfScope() { if (p) p->end(st); }
};
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda):
// a dense float32 tensor of `rank` dims (innermost first), box `box`, zero
// fill outside.
int make_map(CUtensorMap* m, const float* base, int rank, const cuuint64_t* dims,
             const cuuint32_t* box);
bool tma_available();
void workspace_sizes(const pt_plan* plan, size_t* partial_floats, size_t* red_doubles,
                     size_t* image_floats);
int workspace_alloc(const pt_plan* plan, Workspace* ws);
void workspace_free(Workspace* ws);
}  // namespace pt

struct pt_plan {
    int32_t H = 0, W = 0, Z = 1, A = 0, B = 0;
    int32_t row0 = 0, Hg = 0;  // row slab: rows [row0, row0 + H) of an Hg-row image
    double ds = 1.0, h = 1.0;
    std::vector<double> angles;
    std::vector<pt::AngleTab> h_tab;
    pt::AngleTab* d_tab = nullptr;
    int32_t cand_half = 1;     // gather candidates per side: ceil(h/ds) (1 = two-tap)
    int32_t gather_slot = 0;   // floats of staged sinogram per angle in the gather
    int32_t gather_tile = 0;   // index into kGatherTiles
    int32_t fwd_cfg = 0, fwd_ty = 64, fwd_tx = 256;
    int32_t n_bands = 0;
    int32_t max_angles_per_launch = 0;
    pt::Workspace ws;
    int sm_count = 148;
    std::mutex mu;
    std::vector<pt_selection*> selections;
    pt_selection* all = nullptr;
    // (n_subsets, lo, hi) -> (sector selection, subset selections of the sector)
    std::map<std::tuple<int, int, int>,
             std::pair<pt_selection*, std::vector<pt_selection*>>> sector_cache;
};

namespace pt {
// kernels (projector.cu)
void forward_config(int cfg, int32_t* ty, int32_t* tx);
// y = A_S (x - x2) - data_S - data2_S; data / data2 are full sinograms indexed by angle
int launch_forward(pt_plan* plan, Workspace* ws, const pt_selection* sel, const float* x,
                   const float* x2, const float* data, float* y, double* sumsq, cudaStream_t st,
                   const float* data2 = nullptr, double* y64 = nullptr);
// y (float residual rows) = y64 (summed float64 partial line integrals) - data - data2
int launch_forward_finish(pt_plan* plan, const pt_selection* sel, const double* y64,
                          const float* data, const float* data2, float* y, cudaStream_t st);
int launch_adjoint(pt_plan* plan, const pt_selection* sel, const float* y, float* x_out,
                   float alpha, int accumulate, const pt_step_epilogue* ep, cudaStream_t st,
                   Workspace* ws = nullptr, int cat = PT_PROF_GATHER);
int launch_epilogue(pt_plan* plan, const float* g, const pt_step_epilogue* ep, cudaStream_t st);
// fgp.cu
int64_t fgp_workspace_floats(const pt_plan* plan);
int launch_tv_prox(pt_plan* plan, const float* v, double lam, int inner, int nonneg, float* p,
                   float* q, float* w, float* x_out, const float* xhat, float* h,
                   float p_over_gamma, int64_t iteration, int64_t* bad_iter, float* work,
                   cudaStream_t st);
// 3D FGP on z-slabs: a slab owns global planes [z0, z0 + Zl); `work` holds
// fgp3d_slab_floats(Zl, H, W) floats.  ZHalo moves boundary planes between
// ranks: send `count` floats from send_lo to rank - 1 and from send_hi to
// rank + 1, receive into recv_lo from rank - 1 and into recv_hi from rank + 1
// (null pointers skip a direction; ranks 0 / world - 1 have no outer side).
struct Fgp3Slab {
    int Zl = 0, z0 = 0;
    const float* v = nullptr;
    float *p = nullptr, *q = nullptr, *w = nullptr;
    float* x_out = nullptr;
    const float* xhat = nullptr;
    float* h = nullptr;
    float* work = nullptr;
};
struct ZHalo {
    int rank = 0, world = 1;
    void* ctx = nullptr;
    int (*exchange)(void* ctx, const float* send_lo, float* recv_lo, const float* send_hi,
                    float* recv_hi, size_t count, cudaStream_t st) = nullptr;
};
int64_t fgp3d_slab_floats(int Zl, int H, int W);
// 2D row slabs (rows decomposition): slab owns image rows [r0, r0 + Hl)
constexpr int kRowGhost = 9;  // ghost rows per side: the largest FGP T (8) + 1
struct Fgp2Slab {
    int Hl = 0, r0 = 0;
    const float* v = nullptr;  // own rows, Hl x W (as p, q, x_out, xhat, h)
    float *p = nullptr, *q = nullptr;
    float* x_out = nullptr;
    const float* xhat = nullptr;
    float* h = nullptr;
    float* work = nullptr;  // fgp2d_slab_floats(Hl, W)
};
// exchange of the kRowGhost-row boundary bands of n extended arrays (Hl own
// rows between `ghost` ghost rows each side) with the rank -+ 1 slabs
struct RowHalo {
    int rank = 0, world = 1;
    void* ctx = nullptr;
    int (*exchange)(void* ctx, int n, float* const* arrays, int Hl, int W, int ghost,
                    cudaStream_t st) = nullptr;
};
int64_t fgp2d_slab_floats(int Hl, int W);
int fgp2d_rows_run(const Fgp2Slab* slabs, int G, int H, int W, double lam, int inner,
                   int nonneg, float pog, int64_t iteration, int64_t* bad_iter,
                   const RowHalo* halo, cudaStream_t st);
int fgp3d_run(const Fgp3Slab* slabs, int G, int H, int W, int Zg, double lam, int inner,
              int nonneg, float pog, int64_t iteration, int64_t* bad_iter, const ZHalo* halo,
              int sm_count, cudaStream_t st);
// reduce.cu  (out: device doubles, out[0] = result, out[1 .. PT_RED_DOUBLES) scratch)
int launch_dot(const float* a, const float* b, int64_t n, double* out, cudaStream_t st);
int launch_tv_value(const pt_plan* plan, const float* x, double* out, cudaStream_t st);
int launch_diff_norms(const float* x, const float* ref, int64_t n, double* out, cudaStream_t st);
int launch_sum_doubles(const double* in, int64_t n, double* out, int accumulate, cudaStream_t st);
int launch_identity_prox(const float* v, const float* xhat, float* x_out, float* h,
                         float p_over_gamma, int64_t n, int64_t iteration, int64_t* bad_iter,
                         cudaStream_t st);
int launch_scale_by_rsqrt(float* v, const float* u, const double* sumsq, int64_t n,
                          cudaStream_t st);
int launch_fista_momentum(const float* src, const float* x_prev, float* x_out, float* y,
                          float beta, int64_t n, int64_t iteration, int64_t* bad_iter,
                          cudaStream_t st);
int launch_fill_i64(int64_t* p, int64_t value, cudaStream_t st);
}  // namespace pt
