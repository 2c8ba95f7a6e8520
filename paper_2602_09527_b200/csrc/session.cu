// Native executor for the ProxSkip loop: owns the solver state in HBM and
// enqueues whole segments of iterations with no host synchronisation.
//
// One iteration k (pkg/src/proxtomo/solvers.py:189-254):
//   [refresh]  x_snap <- x; G <- A^T(A x_snap - b)           (estimators.py:126-130)
//   forward    r = A_i x - b_i   |   r = A_i (x - x_snap) (SVRG: b cancels)
//   gather     g = A_i^T r, est, base, x_hat, v / x+         (one fused kernel)
//   [theta]    x+ = prox_{(gamma/p) alpha TV}(v), h += (p/gamma)(x+ - x_hat)
// The subset / theta / refresh sequences are drawn on the host with the
// reference's own PCG64 streams (solvers.py:164,174-176) and passed in.
//
// Multi-GPU, three decompositions:
//  * angle sectors (2D): rank g owns angles [g A/G, (g+1) A/G); its
//    forward/gather cover only those rows of subset i; the partial A_i^T r
//    (4 n_px bytes) is summed with ncclAllReduce on the session stream; every
//    rank then applies the identical epilogue and prox (bitwise replicas);
//  * image rows (2D): rank g owns image rows [r0, r0 + Hl) (a row-slab plan);
//    its forward gives partial line integrals of subset i, summed in float64
//    with ncclAllReduce (8 |S_i| B bytes: 0.7 MB at config 2 instead of
//    16 MB), then every rank forms the full residual and gathers, steps and
//    proxes only its own rows (the TV prox exchanges ghost rows with ranks
//    g -+ 1 every launch);
//  * z-slabs (slice-stacked 3D): the projector is slab-local, the 3D prox
//    exchanges ghost planes.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "pt_internal.cuh"

namespace {

// Minimal NCCL ABI (nccl.h, 2.x): resolved at run time from the
// torch-bundled libnccl.so.2 so this library never links a second NCCL.
typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm;
typedef int (*fn_get_uid)(nccl_uid*);
typedef int (*fn_init_rank)(nccl_comm*, int, nccl_uid, int);
typedef int (*fn_allreduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t);
typedef int (*fn_destroy)(nccl_comm);
typedef const char* (*fn_errstr)(int);
typedef int (*fn_p2p)(const void*, size_t, int, int, nccl_comm, cudaStream_t);
typedef int (*fn_bcast)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t);
typedef int (*fn_group)(void);
constexpr int kNcclFloat32 = 7;
constexpr int kNcclFloat64 = 8;
constexpr int kNcclSum = 0;

struct NcclApi {
    void* so = nullptr;
    fn_get_uid get_uid = nullptr;
    fn_init_rank init_rank = nullptr;
    fn_allreduce allreduce = nullptr;
    fn_destroy destroy = nullptr;
    fn_errstr errstr = nullptr;
    fn_p2p send = nullptr, recv = nullptr;  // ncclSend / ncclRecv (z-slab halos)
    fn_bcast bcast = nullptr;               // ncclBroadcast (row gathers of the sharded prox)
    fn_group group_start = nullptr, group_end = nullptr;
};

int nccl_load(const char* path, NcclApi* api)
{
    api->so = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!api->so) {
        pt::set_error("dlopen(%s): %s", path ? path : "libnccl.so.2", dlerror());
        return PT_ENCCL;
    }
    api->get_uid = (fn_get_uid)dlsym(api->so, "ncclGetUniqueId");
    api->init_rank = (fn_init_rank)dlsym(api->so, "ncclCommInitRank");
    api->allreduce = (fn_allreduce)dlsym(api->so, "ncclAllReduce");
    api->destroy = (fn_destroy)dlsym(api->so, "ncclCommDestroy");
    api->errstr = (fn_errstr)dlsym(api->so, "ncclGetErrorString");
    api->send = (fn_p2p)dlsym(api->so, "ncclSend");
    api->recv = (fn_p2p)dlsym(api->so, "ncclRecv");
    api->group_start = (fn_group)dlsym(api->so, "ncclGroupStart");
    api->group_end = (fn_group)dlsym(api->so, "ncclGroupEnd");
    api->bcast = (fn_bcast)dlsym(api->so, "ncclBroadcast");
    if (!api->get_uid || !api->init_rank || !api->allreduce || !api->destroy) {
        pt::set_error("libnccl is missing symbols");
        return PT_ENCCL;
    }
    return PT_OK;
}

}  // namespace

// A process-level NCCL communicator that several sessions can share (one
// ncclCommInitRank per process group instead of one per solve).
struct pt_comm {
    NcclApi api;
    nccl_comm comm = nullptr;
    int rank = 0, world = 1;
};

namespace pt {

cudaEvent_t Profiler::ev()
{
    if (used == pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        pool.push_back(e);
    }
    return pool[used++];
}

void Profiler::begin(int cat, cudaStream_t st)
{
    int rec_cat = -1;
    if (open.empty()) {
        rec_cat = cat;
        outer = cat;
    } else if (outer == PT_PROF_SNAPSHOT && open.size() == 1) {
        if (cat == PT_PROF_FWD_BAND) rec_cat = PT_PROF_SNAP_FWD_BAND;
        else if (cat == PT_PROF_FWD_REDUCE) rec_cat = PT_PROF_SNAP_FWD_REDUCE;
        else if (cat == PT_PROF_GATHER) rec_cat = PT_PROF_SNAP_GATHER;
    }
    if (rec_cat < 0) {
        open.push_back(-1);
        return;
    }
    Rec r{rec_cat, used};
    cudaEventRecord(ev(), st);
    ev();  // reserve the end event
    open.push_back((long)recs.size());
    recs.push_back(r);
}

void Profiler::end(cudaStream_t st)
{
    const long i = open.back();
    open.pop_back();
    if (i >= 0) cudaEventRecord(pool[recs[i].ev0 + 1], st);
    if (open.empty()) outer = -1;
}

int Profiler::collect()
{
    for (const Rec& r : recs) {
        cudaEventSynchronize(pool[r.ev0 + 1]);
        float t = 0.f;
        cudaEventElapsedTime(&t, pool[r.ev0], pool[r.ev0 + 1]);
        ms[r.cat] += t;
        calls[r.cat] += 1;
    }
    recs.clear();
    used = 0;
    return PT_OK;
}

Profiler::~Profiler()
{
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

}  // namespace pt

struct pt_session {
    pt_plan* plan = nullptr;
    pt_solver_desc d{};
    const float* data = nullptr;
    size_t n = 0;
    float* x[2] = {nullptr, nullptr};
    int cur = 0;
    float *h = nullptr, *v = nullptr, *xhat = nullptr;
    float *snap = nullptr, *fg = nullptr;
    float *saga_table = nullptr, *saga_sum = nullptr;
    float *dp = nullptr, *dq = nullptr, *dw = nullptr;
    float* fgp_work = nullptr;
    float* r = nullptr;      // residual rows (largest selection)
    float* rsnap = nullptr;  // SVRG: A x_snap - b over the owned angles (snapshot residual)
    float* g = nullptr;  // partial gradient (multi-GPU)
    float* slab = nullptr;  // backing allocation of the buffers above (+ flag, workspace)
    bool owns_slab = true;  // false: caller-provided memory (pt_session_create_in)
    int64_t* bad = nullptr;
    pt::Workspace ws;
    pt::Profiler prof;
    bool have_duals = false;
    double dual_weight = 0.0;
    double fista_t = 1.0;  // FISTA momentum sequence t_k (solvers.py:384)
    std::vector<pt_selection*> subsets;  // (own rows of) subset i
    pt_selection* own_all = nullptr;     // all (own) angles
    // test hook: G virtual angle sectors on one device (sums what the ranks' allreduce sums)
    int emu = 1;
    std::vector<std::vector<pt_selection*>> emu_subsets;  // [sector][subset]
    std::vector<pt_selection*> emu_all;                    // [sector]
    // NCCL
    NcclApi nccl;
    nccl_comm comm = nullptr;
    bool owns_comm = false;  // created by pt_session_attach_nccl*(), destroyed with the session
    int rank = 0, world = 1;
    // z-slab mode (3D): this rank owns global planes [z0, z0 + Z)
    // of Zg; projector and snapshot are slab-local, the FGP exchanges halos
    bool zslab = false;
    int z0 = 0, Zg = 0;
    float* fgp3_work = nullptr;  // slab FGP workspace (own allocation)
    float* dw_slab = nullptr;    // third dual when the slab plan is 2D (Z = 1)
    pt::ZHalo halo;
    // test hook: G virtual z-slabs of this volume on one device
    int emu_z = 1;
    float* emu_z_work = nullptr;
    // image-rows mode (2D): the plan is rows [plan->row0, + H) of plan->Hg
    bool rows = false;
    double* y64 = nullptr;       // partial line integrals (A rows x B), float64
    float* rows_work = nullptr;  // extended-row FGP state (fgp2d_slab_floats)
    pt::RowHalo rhalo;
    // angle sectors with the 2D TV prox sharded by image rows: rank g runs
    // the prox on rows [sr0, sr0 + sHl) (ghost rows over NCCL, bitwise the
    // whole-image prox) and the new iterate's rows are gathered on every rank
    bool sector_rows = false;
    int sr0 = 0, sHl = 0;
    bool duals_sharded = false;  // dual rows outside [sr0, sr0 + sHl) are stale
};

namespace {

// Selections of angles [lo, hi): subset k = {k, k+N, ...} (geometry.py:75-82)
// restricted to the sector; cached in the plan (a session or a rank reuses them).
int sector_selections(pt_plan* P, int n_subsets, int lo, int hi, pt_selection** all_out,
                      std::vector<pt_selection*>* subs_out)
{
    {
        std::lock_guard<std::mutex> g(P->mu);
        auto it = P->sector_cache.find({n_subsets, lo, hi});
        if (it != P->sector_cache.end()) {
            *all_out = it->second.first;
            *subs_out = it->second.second;
            return PT_OK;
        }
    }
    const int A = P->A;
    pt_selection* all = nullptr;
    std::vector<pt_selection*> subs;
    int rc;
    if (lo == 0 && hi == A) {
        all = P->all;
    } else {
        std::vector<int32_t> own;
        for (int a = lo; a < hi; ++a) own.push_back(a);
        rc = pt_selection_create(P, own.data(), (int32_t)own.size(), &all);
        if (rc) return rc;
    }
    for (int k = 0; k < n_subsets; ++k) {
        std::vector<int32_t> idx;
        for (int a = k; a < A; a += n_subsets)
            if (a >= lo && a < hi) idx.push_back(a);
        pt_selection* sel = nullptr;
        rc = pt_selection_create(P, idx.data(), (int32_t)idx.size(), &sel);
        if (rc) return rc;
        subs.push_back(sel);
    }
    {
        std::lock_guard<std::mutex> g(P->mu);
        P->sector_cache[{n_subsets, lo, hi}] = {all, subs};
    }
    *all_out = all;
    *subs_out = subs;
    return PT_OK;
}

// Estimators whose step uses every (owned) angle: the full gradient and FISTA.
bool full_kind(int est) { return est == PT_EST_FULL || est == PT_EST_FISTA; }

// First owned angle: the sector start in the angle-sector layout; 0 in the
// slab layouts (rows / z-slabs own every angle, build_selections).
int owned_angle_lo(const pt_session* s)
{
    if (s->zslab || s->rows) return 0;
    return (int)((long long)s->plan->A * s->rank / s->world);
}

int build_selections(pt_session* s)
{
    pt_plan* P = s->plan;
    const int A = P->A;
    const bool all = s->zslab || s->rows;  // slab modes own every angle
    const int world = all ? 1 : s->world, rank = all ? 0 : s->rank;
    const int lo = owned_angle_lo(s);
    const int hi = (int)((long long)A * (rank + 1) / world);
    const int n = !full_kind(s->d.estimator) ? s->d.n_subsets : 0;
    return sector_selections(P, n, lo, hi, &s->own_all, &s->subsets);
}

int allreduce(pt_session* s, float* buf, cudaStream_t st)
{
    if (!s->comm || s->zslab || s->rows) return PT_OK;
    int e = s->nccl.allreduce(buf, buf, s->n, kNcclFloat32, kNcclSum, s->comm, st);
    if (e != 0) {
        pt::set_error("ncclAllReduce: %s", s->nccl.errstr ? s->nccl.errstr(e) : "error");
        return PT_ENCCL;
    }
    return PT_OK;
}

// Rows mode: residual rows of `sel` = (sum over ranks of the slabs' partial
// line integrals) - data - data2; the float64 sum is one ncclAllReduce.
int rows_forward(pt_session* s, const pt_selection* sel, const float* x, const float* data2,
                 float* out, cudaStream_t st)
{
    pt_plan* P = s->plan;
    int rc = pt::launch_forward(P, &s->ws, sel, x, nullptr, nullptr, nullptr, nullptr, st,
                                nullptr, s->y64);
    if (rc || sel->n == 0) return rc;
    {
        pt::ProfScope ps(&s->ws, PT_PROF_OTHER, st);
        const int e = s->nccl.allreduce(s->y64, s->y64, (size_t)sel->n * P->Z * P->B,
                                        kNcclFloat64, kNcclSum, s->comm, st);
        if (e != 0) {
            pt::set_error("ncclAllReduce: %s", s->nccl.errstr ? s->nccl.errstr(e) : "error");
            return PT_ENCCL;
        }
    }
    return pt::launch_forward_finish(P, sel, s->y64, s->data, data2, out, st);
}

// G = A^T (A x - b) over the owned angles, summed over ranks (estimators.py:40-48).
// The residual A x - b is kept in `res` (SVRG: the snapshot residual, so each
// step's A_i(x - x_snap) = (A_i x - b_i) - (A_i x_snap - b_i) needs one
// projection of x only; the subtraction is done in float64 in the reduction).
int full_gradient(pt_session* s, const float* x, float* out, float* res, cudaStream_t st)
{
    pt::ProfScope ps(&s->ws, PT_PROF_SNAPSHOT, st);
    pt_plan* P = s->plan;
    int rc = s->rows ? rows_forward(s, s->own_all, x, nullptr, res, st)
                     : pt::launch_forward(P, &s->ws, s->own_all, x, nullptr, s->data, res,
                                          nullptr, st);
    if (rc) return rc;
    if (s->emu > 1) {
        // virtual sectors: each sector's A_S^T over the shared residual, summed
        for (int g = 0; g < s->emu; ++g) {
            const pt_selection* sg = s->emu_all[g];
            if (sg->n == 0) {
                if (g == 0) PT_CHECK_CUDA(cudaMemsetAsync(out, 0, s->n * 4, st));
                continue;
            }
            // the residual rows of sector g start at its first angle
            const size_t off = (size_t)sg->h_angle[0] * P->Z * P->B;
            rc = pt::launch_adjoint(P, sg, res + off, out, 1.f, g > 0, nullptr, st, &s->ws);
            if (rc) return rc;
        }
        return PT_OK;
    }
    if (s->own_all->n == 0) {
        PT_CHECK_CUDA(cudaMemsetAsync(out, 0, s->n * 4, st));
    } else {
        rc = pt::launch_adjoint(P, s->own_all, res, out, 1.f, 0, nullptr, st, &s->ws);
        if (rc) return rc;
    }
    return allreduce(s, out, st);
}

// The snapshot residual indexed by geometry angle (rows [lo, hi) are owned).
const float* rsnap_by_angle(const pt_session* s)
{
    return s->rsnap - (ptrdiff_t)owned_angle_lo(s) * s->plan->Z * s->plan->B;
}

// Halo exchange with the z-neighbours (ncclSend / ncclRecv in one group).
int nccl_halo(void* ctx, const float* send_lo, float* recv_lo, const float* send_hi,
              float* recv_hi, size_t count, cudaStream_t st)
{
    pt_session* s = (pt_session*)ctx;
    const NcclApi& api = s->nccl;
    const bool lo = s->rank > 0, hi = s->rank + 1 < s->world;
    int e = api.group_start();
    if (!e && lo && send_lo) e = api.send(send_lo, count, kNcclFloat32, s->rank - 1, s->comm, st);
    if (!e && lo && recv_lo) e = api.recv(recv_lo, count, kNcclFloat32, s->rank - 1, s->comm, st);
    if (!e && hi && send_hi) e = api.send(send_hi, count, kNcclFloat32, s->rank + 1, s->comm, st);
    if (!e && hi && recv_hi) e = api.recv(recv_hi, count, kNcclFloat32, s->rank + 1, s->comm, st);
    const int e2 = api.group_end();
    if (e || e2) {
        pt::set_error("NCCL halo exchange: %s", api.errstr ? api.errstr(e ? e : e2) : "error");
        return PT_ENCCL;
    }
    return PT_OK;
}

// Ghost-row exchange of a rows rank with ranks -+ 1 (one NCCL group for all
// n arrays; arrays hold `ghost` rows, Hl own rows, `ghost` rows).
int nccl_rows_halo(void* ctx, int n, float* const* arrays, int Hl, int W, int ghost,
                   cudaStream_t st)
{
    pt_session* s = (pt_session*)ctx;
    const NcclApi& api = s->nccl;
    const bool lo = s->rank > 0, hi = s->rank + 1 < s->world;
    const size_t cnt = (size_t)ghost * W;
    int e = api.group_start();
    for (int i = 0; i < n && !e; ++i) {
        float* a = arrays[i];
        if (lo && !e) e = api.send(a + cnt, cnt, kNcclFloat32, s->rank - 1, s->comm, st);
        if (lo && !e) e = api.recv(a, cnt, kNcclFloat32, s->rank - 1, s->comm, st);
        if (hi && !e) e = api.send(a + (size_t)Hl * W, cnt, kNcclFloat32, s->rank + 1, s->comm, st);
        if (hi && !e) e = api.recv(a + (size_t)(ghost + Hl) * W, cnt, kNcclFloat32, s->rank + 1,
                                   s->comm, st);
    }
    const int e2 = api.group_end();
    if (e || e2) {
        pt::set_error("NCCL row halo exchange: %s", api.errstr ? api.errstr(e ? e : e2) : "error");
        return PT_ENCCL;
    }
    return PT_OK;
}

// The 2D TV prox of a rows rank: its own rows, ghost rows over NCCL.
int rows_tv_prox(pt_session* s, double lam, float pog, float* xn, int64_t k, cudaStream_t st)
{
    pt_plan* P = s->plan;
    pt::Fgp2Slab a;
    a.Hl = P->H; a.r0 = P->row0;
    a.v = s->v; a.p = s->dp; a.q = s->dq;
    a.x_out = xn; a.xhat = s->xhat; a.h = s->h; a.work = s->rows_work;
    return pt::fgp2d_rows_run(&a, 1, P->Hg, P->W, lam, s->d.tv_inner, s->d.tv_nonneg, pog, k,
                              s->bad, &s->rhalo, st);
}

// Rows [H g / G, H (g + 1) / G) of rank g (the image-row split of the sector
// layout's sharded prox; distributed.rowslab_bounds uses the same formula).
inline int sector_row(int H, int g, int world) { return (int)((long long)H * g / world); }

// Every rank's rows of `a` (H x W, rank g's rows valid on rank g) on every
// rank: one grouped ncclBroadcast per owner, in place.
int gather_sector_rows(pt_session* s, float* a, cudaStream_t st)
{
    const NcclApi& api = s->nccl;
    const int H = s->plan->H, W = s->plan->W;
    int e = api.group_start();
    for (int g = 0; g < s->world && !e; ++g) {
        const int r0 = sector_row(H, g, s->world), r1 = sector_row(H, g + 1, s->world);
        float* rows = a + (size_t)r0 * W;
        e = api.bcast(rows, rows, (size_t)(r1 - r0) * W, kNcclFloat32, g, s->comm, st);
    }
    const int e2 = api.group_end();
    if (e || e2) {
        pt::set_error("NCCL row gather: %s", api.errstr ? api.errstr(e ? e : e2) : "error");
        return PT_ENCCL;
    }
    return PT_OK;
}

// The 2D TV prox of an angle-sector rank, sharded by image rows: the rows
// FGP driver on this rank's rows of the (replicated) image -- ghost rows from
// ranks g -+ 1, bitwise the whole-image prox -- then the new iterate and the
// control variate rows gathered on every rank.  The dual state keeps only the
// own rows current (gathered at the end of a run call, see pt_session_run).
// FISTA (fista = true): x+ = prox(v) only -- no control variate, and the
// momentum kernel checks x+ for finiteness.
int sector_rows_tv_prox(pt_session* s, double lam, float pog, float* xn, int64_t k,
                        cudaStream_t st, bool fista)
{
    pt_plan* P = s->plan;
    const size_t off = (size_t)s->sr0 * P->W;
    pt::Fgp2Slab a;
    a.Hl = s->sHl; a.r0 = s->sr0;
    a.v = s->v + off; a.p = s->dp + off; a.q = s->dq + off;
    a.x_out = xn + off; a.work = s->rows_work;
    a.xhat = fista ? nullptr : s->xhat + off;
    a.h = fista ? nullptr : s->h + off;
    int rc = pt::fgp2d_rows_run(&a, 1, P->H, P->W, lam, s->d.tv_inner, s->d.tv_nonneg,
                                fista ? 0.f : pog, k, fista ? nullptr : s->bad, &s->rhalo, st);
    s->duals_sharded = true;
    if (!rc) rc = gather_sector_rows(s, xn, st);
    if (!rc && !fista) rc = gather_sector_rows(s, s->h, st);
    return rc;
}

// The 3D TV prox of a z-slab rank (halos over NCCL), or of G virtual slabs of
// this volume on one device (halos by device copies).
int slab_tv_prox(pt_session* s, double lam, float pog, float* xn, int64_t k, cudaStream_t st)
{
    pt_plan* P = s->plan;
    const size_t HW = (size_t)P->H * P->W;
    float* dw = s->dw ? s->dw : s->dw_slab;
    std::vector<pt::Fgp3Slab> sl;
    if (s->zslab) {
        pt::Fgp3Slab a;
        a.Zl = P->Z; a.z0 = s->z0;
        a.v = s->v; a.p = s->dp; a.q = s->dq; a.w = dw;
        a.x_out = xn; a.xhat = s->xhat; a.h = s->h; a.work = s->fgp3_work;
        sl.push_back(a);
    } else {
        float* work = s->emu_z_work;
        for (int g = 0; g < s->emu_z; ++g) {
            const int za = (int)((long long)P->Z * g / s->emu_z);
            const int zb = (int)((long long)P->Z * (g + 1) / s->emu_z);
            const size_t off = (size_t)za * HW;
            pt::Fgp3Slab a;
            a.Zl = zb - za; a.z0 = za;
            a.v = s->v + off; a.p = s->dp + off; a.q = s->dq + off; a.w = dw + off;
            a.x_out = xn + off; a.xhat = s->xhat + off; a.h = s->h + off; a.work = work;
            work += pt::fgp3d_slab_floats(a.Zl, P->H, P->W);
            sl.push_back(a);
        }
    }
    const int Zg = s->zslab ? s->Zg : P->Z;
    return pt::fgp3d_run(sl.data(), (int)sl.size(), P->H, P->W, Zg, lam, s->d.tv_inner,
                         s->d.tv_nonneg, pog, k, s->bad, s->zslab ? &s->halo : nullptr,
                         P->sm_count, st);
}

}  // namespace

extern "C" {

namespace {

int check_desc(const pt_plan* plan, const pt_solver_desc* desc)
{
    if (!(desc->gamma > 0.0)) { pt::set_error("gamma must be positive"); return PT_EINVAL; }
    if (!(desc->skip_probability > 0.0 && desc->skip_probability <= 1.0)) {
        pt::set_error("skip_probability must be in (0, 1]");
        return PT_EINVAL;
    }
    if (desc->estimator < PT_EST_FULL || desc->estimator > PT_EST_FISTA) { pt::set_error("unknown estimator"); return PT_EINVAL; }
    if (desc->estimator == PT_EST_FISTA && desc->skip_probability != 1.0) {
        pt::set_error("FISTA applies the prox every iteration (skip_probability 1)");
        return PT_EINVAL;
    }
    if (!full_kind(desc->estimator) && (desc->n_subsets < 1 || desc->n_subsets > plan->A)) {
        pt::set_error("n_subsets must be in [1, n_angles], got %d for %d angles", desc->n_subsets, plan->A);
        return PT_EINVAL;
    }
    if (desc->prox_kind == 1 && (!(desc->tv_alpha > 0.0) || desc->tv_inner < 1)) {
        pt::set_error("bad TV configuration");
        return PT_EINVAL;
    }
    return PT_OK;
}

// Carve every session buffer out of one allocation (256-byte aligned
// pieces): the state, the divergence flag and the projector workspace.
// base == nullptr: only count.  Returns the bytes needed.
size_t session_layout(const pt_plan* plan, const pt_solver_desc* desc, pt_session* s, char* base)
{
    const size_t n = (size_t)plan->Z * plan->H * plan->W;
    const size_t sino = (size_t)plan->A * plan->Z * plan->B;
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
        char* p = base ? base + off : nullptr;
        off += (std::max<size_t>(bytes, 1) + 255) & ~size_t(255);
        return p;
    };
    auto F = [&](float** dst, size_t cnt) {
        char* p = take(cnt * sizeof(float));
        if (dst) *dst = (float*)p;
    };
    const bool vr = desc->estimator == PT_EST_SVRG || desc->estimator == PT_EST_LSVRG;
    F(s ? &s->x[0] : nullptr, n); F(s ? &s->x[1] : nullptr, n);
    F(s ? &s->h : nullptr, n); F(s ? &s->v : nullptr, n); F(s ? &s->xhat : nullptr, n);
    if (vr) { F(s ? &s->snap : nullptr, n); F(s ? &s->fg : nullptr, n); F(s ? &s->rsnap : nullptr, sino); }
    if (desc->estimator == PT_EST_FISTA) F(s ? &s->snap : nullptr, n);  // momentum point y
    if (desc->estimator == PT_EST_SAGA) {
        F(s ? &s->saga_table : nullptr, n * desc->n_subsets);
        F(s ? &s->saga_sum : nullptr, n);
    }
    if (desc->prox_kind == 1) {
        F(s ? &s->dp : nullptr, n); F(s ? &s->dq : nullptr, n);
        if (plan->Z > 1) F(s ? &s->dw : nullptr, n);
        F(s ? &s->fgp_work : nullptr, (size_t)pt::fgp_workspace_floats(plan));
    }
    F(s ? &s->r : nullptr, sino);
    F(s ? &s->g : nullptr, n);
    {
        char* p = take(sizeof(int64_t));
        if (s) s->bad = (int64_t*)p;
    }
    // projector workspace (band partials, reduction scratch, image temp)
    size_t pf, rd, imf;
    pt::workspace_sizes(plan, &pf, &rd, &imf);
    {
        char* a = take(pf * sizeof(float));
        char* b = take(rd * sizeof(double));
        char* c = take(imf * sizeof(float));
        if (s) {
            s->ws.partial = (float*)a; s->ws.partial_floats = pf;
            s->ws.red = (double*)b; s->ws.red_doubles = rd;
            s->ws.image = (float*)c; s->ws.image_floats = imf;
        }
    }
    return off;
}

}  // namespace

int64_t pt_session_workspace_bytes(pt_plan* plan, const pt_solver_desc* desc)
{
    if (!plan || !desc) { pt::set_error("null argument"); return -1; }
    return (int64_t)session_layout(plan, desc, nullptr, nullptr);
}

int pt_session_create_in(pt_plan* plan, const pt_solver_desc* desc, const float* data,
                         const float* x0, void* workspace, int64_t workspace_bytes,
                         pt_session** out, void* stream)
{
    if (!plan || !desc || !data || !out) { pt::set_error("null argument"); return PT_EINVAL; }
    int rc = check_desc(plan, desc);
    if (rc) return rc;
    const size_t need = session_layout(plan, desc, nullptr, nullptr);
    if (workspace && (workspace_bytes < 0 || (size_t)workspace_bytes < need ||
                      ((uintptr_t)workspace & 255))) {
        pt::set_error("session workspace: need %zu bytes, 256-byte aligned", need);
        return PT_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    pt_session* s = new pt_session();
    s->plan = plan;
    s->d = *desc;
    s->data = data;
    s->n = (size_t)plan->Z * plan->H * plan->W;
    const size_t n = s->n;
    char* base = (char*)workspace;
    if (!base) {
        if (cudaMalloc(&base, need) != cudaSuccess) {
            pt::set_error("session allocation of %zu bytes failed", need);
            delete s;
            return PT_ECUDA;
        }
        s->owns_slab = true;
    } else {
        s->owns_slab = false;
    }
    s->slab = (float*)base;
    session_layout(plan, desc, s, base);
    s->ws.prof = &s->prof;
    rc = build_selections(s);
    if (rc == PT_OK) {
        // solvers.py:161,172,178-179: x0 (or zeros), h = 0, SAGA table/sum = 0
        if (x0) rc = cudaMemcpyAsync(s->x[0], x0, n * 4, cudaMemcpyDeviceToDevice, st) ? PT_ECUDA : PT_OK;
        else rc = cudaMemsetAsync(s->x[0], 0, n * 4, st) ? PT_ECUDA : PT_OK;
        if (!rc) rc = cudaMemsetAsync(s->h, 0, n * 4, st) ? PT_ECUDA : PT_OK;
        if (!rc && s->saga_table) rc = cudaMemsetAsync(s->saga_table, 0, n * 4 * desc->n_subsets, st) ? PT_ECUDA : PT_OK;
        if (!rc && s->saga_sum) rc = cudaMemsetAsync(s->saga_sum, 0, n * 4, st) ? PT_ECUDA : PT_OK;
        if (!rc) rc = pt::launch_fill_i64(s->bad, INT64_MAX, st);
    }
    if (rc != PT_OK) {
        pt_session_destroy(s);
        return rc;
    }
    *out = s;
    return PT_OK;
}

int pt_session_create(pt_plan* plan, const pt_solver_desc* desc, const float* data,
                      const float* x0, pt_session** out, void* stream)
{
    return pt_session_create_in(plan, desc, data, x0, nullptr, 0, out, stream);
}

int pt_session_destroy(pt_session* s)
{
    if (!s) return PT_OK;
    cudaDeviceSynchronize();
    if (s->slab && s->owns_slab) cudaFree(s->slab);  // state, flag and workspace
    if (s->comm && s->owns_comm && s->nccl.destroy) s->nccl.destroy(s->comm);
    if (s->fgp3_work) cudaFree(s->fgp3_work);
    if (s->dw_slab) cudaFree(s->dw_slab);
    if (s->emu_z_work) cudaFree(s->emu_z_work);
    if (s->y64) cudaFree(s->y64);
    if (s->rows_work) cudaFree(s->rows_work);
    delete s;
    return PT_OK;
}

int pt_session_init(pt_session* s, void* stream)
{
    if (!s) { pt::set_error("null session"); return PT_EINVAL; }
    cudaStream_t st = (cudaStream_t)stream;
    if (s->d.estimator == PT_EST_FISTA) {
        // run_fista (solvers.py:378): y = x0, t = 1
        s->fista_t = 1.0;
        PT_CHECK_CUDA(cudaMemcpyAsync(s->snap, s->x[s->cur], s->n * 4, cudaMemcpyDeviceToDevice, st));
        return PT_OK;
    }
    if (s->d.estimator != PT_EST_SVRG && s->d.estimator != PT_EST_LSVRG) return PT_OK;
    // init_svrg_state (estimators.py:117-123): snapshot = x0, G = full gradient
    PT_CHECK_CUDA(cudaMemcpyAsync(s->snap, s->x[s->cur], s->n * 4, cudaMemcpyDeviceToDevice, st));
    return full_gradient(s, s->snap, s->fg, s->rsnap, st);
}

int pt_session_run(pt_session* s, int32_t n_steps, const int32_t* host_subset,
                   const uint8_t* host_theta, const uint8_t* host_refresh, int64_t k0, void* stream)
{
    if (!s || n_steps < 0) { pt::set_error("bad argument"); return PT_EINVAL; }
    cudaStream_t st = (cudaStream_t)stream;
    pt_plan* P = s->plan;
    const pt_solver_desc& d = s->d;
    const bool vr = (d.estimator == PT_EST_SVRG || d.estimator == PT_EST_LSVRG);
    const bool fista = d.estimator == PT_EST_FISTA;
    if (fista && (s->zslab || s->rows)) {
        pt::set_error("FISTA runs on one device or angle sectors");
        return PT_EINVAL;
    }
    const double gamma = d.gamma, p = d.skip_probability;
    for (int j = 0; j < n_steps; ++j) {
        const int64_t k = k0 + j;
        int rc = PT_OK;
        const bool refreshed = vr && host_refresh && host_refresh[j];
        if (refreshed) {
            // refresh_svrg_state (estimators.py:126-130)
            {
                pt::ProfScope ps(&s->ws, PT_PROF_OTHER, st);
                PT_CHECK_CUDA(cudaMemcpyAsync(s->snap, s->x[s->cur], s->n * 4, cudaMemcpyDeviceToDevice, st));
            }
            rc = full_gradient(s, s->snap, s->fg, s->rsnap, st);
            if (rc) return rc;
        }
        const pt_selection* sel = s->own_all;
        int i = 0;
        if (!full_kind(d.estimator)) {
            i = host_subset ? host_subset[j] : 0;
            if (i < 0 || i >= d.n_subsets) {
                pt::set_error("subset index %d out of range [0, %d)", i, d.n_subsets);
                return PT_EINVAL;
            }
            sel = s->subsets[i];
        }
        const float* xc = s->x[s->cur];
        float* xn = s->x[1 - s->cur];
        // the point the gradient is taken at: x, or FISTA's momentum point y
        const float* xg = fista ? s->snap : xc;
        const int theta = (p >= 1.0) ? 1 : (host_theta ? host_theta[j] : 0);

        // Right after a refresh x == x_snap bitwise, so the reference's
        // N (g_i(x) - g_i(x_snap)) is exactly 0 (two identical float64
        // evaluations) and the estimate is the snapshot gradient itself: no
        // subset projection, the epilogue runs on a zero difference.
        // forward: residual rows of the (own part of the) selection
        if (refreshed || s->emu > 1)
            ;  // none / per virtual sector below
        else if (s->rows)
            rc = rows_forward(s, sel, xc, vr ? rsnap_by_angle(s) : nullptr, s->r, st);
        else if (vr)  // A_i (x - x_snap) = (A_i x - b_i) - (A_i x_snap - b_i)
            rc = pt::launch_forward(P, &s->ws, sel, xc, nullptr, s->data, s->r, nullptr, st,
                                    rsnap_by_angle(s));
        else
            rc = pt::launch_forward(P, &s->ws, sel, xg, nullptr, s->data, s->r, nullptr, st);
        if (rc) return rc;

        pt_step_epilogue ep;
        memset(&ep, 0, sizeof(ep));
        ep.estimator = fista ? PT_EST_FULL : d.estimator;
        ep.theta = theta;
        ep.n_scale = (float)d.n_subsets;
        ep.gamma = (float)gamma;
        ep.hcoef = (float)(gamma - gamma / p);  // solvers.py:242, exactly 0 at p = 1
        ep.iteration = k;
        ep.x = xg;
        ep.h = s->h;
        if (d.estimator == PT_EST_SAGA) {
            ep.aux0 = s->saga_table + (size_t)i * s->n;
            ep.aux1 = s->saga_sum;
        } else if (vr) {
            ep.aux0 = s->fg;
        }
        ep.x_out = xn;
        ep.v_out = s->v;
        ep.xhat_out = s->xhat;
        ep.bad_iter = s->bad;
        if (refreshed) {
            pt::ProfScope ps(&s->ws, PT_PROF_OTHER, st);
            rc = pt::launch_epilogue(P, nullptr, &ep, st);
        } else if (s->emu > 1) {
            // virtual ranks: partial A_i^T r per sector, summed in g, then the epilogue
            for (int g = 0; g < s->emu && !rc; ++g) {
                const pt_selection* sg = full_kind(d.estimator) ? s->emu_all[g]
                                                                : s->emu_subsets[g][i];
                if (sg->n == 0) {
                    if (g == 0) PT_CHECK_CUDA(cudaMemsetAsync(s->g, 0, s->n * 4, st));
                    continue;
                }
                if (vr)
                    rc = pt::launch_forward(P, &s->ws, sg, xc, nullptr, s->data, s->r, nullptr, st,
                                            rsnap_by_angle(s));
                else
                    rc = pt::launch_forward(P, &s->ws, sg, xg, nullptr, s->data, s->r, nullptr, st);
                if (!rc) rc = pt::launch_adjoint(P, sg, s->r, s->g, 1.f, g > 0, nullptr, st, &s->ws);
            }
            if (!rc) rc = pt::launch_epilogue(P, s->g, &ep, st);
        } else if (!s->comm || s->zslab || s->rows) {
            rc = pt::launch_adjoint(P, sel, s->r, nullptr, 1.f, 0, &ep, st, &s->ws);
        } else {
            if (sel->n == 0) {
                PT_CHECK_CUDA(cudaMemsetAsync(s->g, 0, s->n * 4, st));
            } else {
                rc = pt::launch_adjoint(P, sel, s->r, s->g, 1.f, 0, nullptr, st, &s->ws);
            }
            pt::ProfScope ps(&s->ws, PT_PROF_OTHER, st);
            if (!rc) rc = allreduce(s, s->g, st);
            if (!rc) rc = pt::launch_epilogue(P, s->g, &ep, st);
        }
        if (rc) return rc;

        if (theta) {
            const float pog = (float)(p / gamma);
            if (d.prox_kind == 1) {
                // _apply_prox -> tv_prox with tau = gamma/p (solvers.py:217-223,242-243)
                const double lam = (gamma / p) * d.tv_alpha;
                const bool warm = d.tv_warm_start && s->have_duals &&
                                  fabs(s->dual_weight - lam) <= 1e-12 * fabs(lam);
                pt::ProfScope ps(&s->ws, PT_PROF_FGP, st);
                float* dw = s->dw ? s->dw : s->dw_slab;
                if (!warm) {
                    PT_CHECK_CUDA(cudaMemsetAsync(s->dp, 0, s->n * 4, st));
                    PT_CHECK_CUDA(cudaMemsetAsync(s->dq, 0, s->n * 4, st));
                    if (dw) PT_CHECK_CUDA(cudaMemsetAsync(dw, 0, s->n * 4, st));
                }
                if (fista && s->sector_rows)
                    rc = sector_rows_tv_prox(s, lam, pog, xn, k, st, true);
                else if (fista)  // x+ = prox(v); no control variate (the momentum kernel checks x+)
                    rc = pt::launch_tv_prox(P, s->v, lam, d.tv_inner, d.tv_nonneg, s->dp, s->dq,
                                            s->dw, xn, nullptr, nullptr, 0.f, k, nullptr,
                                            s->fgp_work, st);
                else if (s->zslab || s->emu_z > 1)
                    rc = slab_tv_prox(s, lam, pog, xn, k, st);
                else if (s->rows)
                    rc = rows_tv_prox(s, lam, pog, xn, k, st);
                else if (s->sector_rows)
                    rc = sector_rows_tv_prox(s, lam, pog, xn, k, st, false);
                else
                    rc = pt::launch_tv_prox(P, s->v, lam, d.tv_inner, d.tv_nonneg, s->dp, s->dq,
                                            s->dw, xn, s->xhat, s->h, pog, k, s->bad,
                                            s->fgp_work, st);
                s->have_duals = true;
                s->dual_weight = lam;
            } else if (!fista) {
                pt::ProfScope ps(&s->ws, PT_PROF_OTHER, st);
                rc = pt::launch_identity_prox(s->v, s->xhat, xn, s->h, pog, (int64_t)s->n, k,
                                              s->bad, st);
            }
            if (rc) return rc;
        }
        if (fista) {
            // solvers.py:384-386: t_next, y = x+ + ((t - 1) / t_next)(x+ - x)
            const double t = s->fista_t;
            const double t_next = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
            s->fista_t = t_next;
            pt::ProfScope ps(&s->ws, PT_PROF_OTHER, st);
            rc = pt::launch_fista_momentum(d.prox_kind == 1 ? xn : s->v, xc, xn, s->snap,
                                           (float)((t - 1.0) / t_next), (int64_t)s->n, k, s->bad,
                                           st);
            if (rc) return rc;
        }
        s->cur = 1 - s->cur;
    }
    if (s->duals_sharded) {
        // sharded sector prox: whole dual images at the API boundary (the
        // state views, the next call's warm start reads only its own rows)
        int rc = gather_sector_rows(s, s->dp, st);
        if (!rc) rc = gather_sector_rows(s, s->dq, st);
        if (rc) return rc;
        s->duals_sharded = false;
    }
    return PT_OK;
}

int pt_session_run_marked(pt_session* s, int32_t n_steps, const int32_t* host_subset,
                          const uint8_t* host_theta, const uint8_t* host_refresh, int64_t k0,
                          int32_t n_marks, const int32_t* host_marks, void* const* events,
                          void* stream)
{
    if (!s || n_steps < 0 || n_marks < 0 || (n_marks && (!host_marks || !events))) {
        pt::set_error("bad argument");
        return PT_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    int32_t done = 0;
    for (int32_t m = 0; m < n_marks; ++m) {
        const int32_t upto = host_marks[m];
        if (upto < done || upto > n_steps) { pt::set_error("marks must ascend within the steps"); return PT_EINVAL; }
        const int rc = pt_session_run(s, upto - done, host_subset ? host_subset + done : nullptr,
                                      host_theta ? host_theta + done : nullptr,
                                      host_refresh ? host_refresh + done : nullptr, k0 + done,
                                      stream);
        if (rc) return rc;
        PT_CHECK_CUDA(cudaEventRecord((cudaEvent_t)events[m], st));
        done = upto;
    }
    if (done < n_steps)
        return pt_session_run(s, n_steps - done, host_subset ? host_subset + done : nullptr,
                              host_theta ? host_theta + done : nullptr,
                              host_refresh ? host_refresh + done : nullptr, k0 + done, stream);
    return PT_OK;
}

int pt_session_set_profiling(pt_session* s, int32_t on)
{
    if (!s) { pt::set_error("null session"); return PT_EINVAL; }
    s->prof.on = on != 0;
    return PT_OK;
}

int pt_session_profile(pt_session* s, double* host_ms, int64_t* host_calls)
{
    if (!s || !host_ms || !host_calls) { pt::set_error("null argument"); return PT_EINVAL; }
    s->prof.collect();
    for (int c = 0; c < PT_PROF_N; ++c) {
        host_ms[c] = s->prof.ms[c];
        host_calls[c] = s->prof.calls[c];
        s->prof.ms[c] = 0.0;
        s->prof.calls[c] = 0;
    }
    return PT_OK;
}

float* pt_session_x(pt_session* s) { return s ? s->x[s->cur] : nullptr; }
float* pt_session_h(pt_session* s) { return s ? s->h : nullptr; }
int64_t* pt_session_bad_iter(pt_session* s) { return s ? s->bad : nullptr; }

float* pt_session_buffer(pt_session* s, int32_t which)
{
    if (!s) return nullptr;
    switch (which) {
        case 0: return s->snap;
        case 1: return s->fg;
        case 2: return s->saga_sum;
        case 3: return s->saga_table;
        case 4: return s->dp;
        case 5: return s->dq;
        case 6: return s->dw ? s->dw : s->dw_slab;
        default: return nullptr;
    }
}

int pt_nccl_unique_id(const char* nccl_path, uint8_t* host_out128)
{
    NcclApi api;
    int rc = nccl_load(nccl_path, &api);
    if (rc) return rc;
    nccl_uid id;
    int e = api.get_uid(&id);
    if (e != 0) { pt::set_error("ncclGetUniqueId failed (%d)", e); return PT_ENCCL; }
    memcpy(host_out128, id.internal, 128);
    return PT_OK;
}

int pt_session_emulate_sectors(pt_session* s, int32_t world)
{
    if (!s || world < 1) { pt::set_error("bad argument"); return PT_EINVAL; }
    if (s->comm) { pt::set_error("session already attached to NCCL"); return PT_EINVAL; }
    pt_plan* P = s->plan;
    const int A = P->A;
    s->emu_subsets.assign(world, {});
    s->emu_all.assign(world, nullptr);
    const int n = !full_kind(s->d.estimator) ? s->d.n_subsets : 0;
    for (int g = 0; g < world; ++g) {
        const int lo = (int)((long long)A * g / world), hi = (int)((long long)A * (g + 1) / world);
        int rc = sector_selections(P, n, lo, hi, &s->emu_all[g], &s->emu_subsets[g]);
        if (rc) return rc;
    }
    s->emu = world;
    return PT_OK;
}

int pt_session_emulate_zslabs(pt_session* s, int32_t slabs)
{
    if (!s || slabs < 1) { pt::set_error("bad argument"); return PT_EINVAL; }
    if (s->comm) { pt::set_error("session already attached to NCCL"); return PT_EINVAL; }
    pt_plan* P = s->plan;
    if (slabs > P->Z) { pt::set_error("more slabs (%d) than slices (%d)", slabs, P->Z); return PT_EINVAL; }
    if (s->d.prox_kind != 1) { pt::set_error("z-slabs only change the TV prox"); return PT_EINVAL; }
    int64_t total = 0;
    for (int g = 0; g < slabs; ++g) {
        const int za = (int)((long long)P->Z * g / slabs), zb = (int)((long long)P->Z * (g + 1) / slabs);
        total += pt::fgp3d_slab_floats(zb - za, P->H, P->W);
    }
    if (s->emu_z_work) cudaFree(s->emu_z_work);
    s->emu_z_work = nullptr;
    PT_CHECK_CUDA(cudaMalloc(&s->emu_z_work, (size_t)total * sizeof(float)));
    s->emu_z = slabs;
    return PT_OK;
}

int pt_nccl_comm_create(const char* nccl_path, const uint8_t* host_id128, int32_t rank,
                        int32_t world, pt_comm** out)
{
    if (!host_id128 || !out || world < 1 || rank < 0 || rank >= world) { pt::set_error("bad argument"); return PT_EINVAL; }
    pt_comm* c = new pt_comm();
    int rc = nccl_load(nccl_path, &c->api);
    if (rc) { delete c; return rc; }
    nccl_uid id;
    memcpy(id.internal, host_id128, 128);
    int e = c->api.init_rank(&c->comm, world, id, rank);
    if (e != 0) {
        pt::set_error("ncclCommInitRank failed (%d)", e);
        delete c;
        return PT_ENCCL;
    }
    c->rank = rank;
    c->world = world;
    *out = c;
    return PT_OK;
}

int pt_nccl_comm_destroy(pt_comm* c)
{
    if (!c) return PT_OK;
    cudaDeviceSynchronize();
    if (c->comm && c->api.destroy) c->api.destroy(c->comm);
    delete c;
    return PT_OK;
}

namespace {

int attach_sector(pt_session* s, const NcclApi& api, nccl_comm comm, int rank, int world)
{
    s->nccl = api;
    s->comm = comm;
    s->rank = rank;
    s->world = world;
    pt_plan* P = s->plan;
    // the replicated TV prox is sharded by image rows when every rank gets
    // enough rows for the ghost exchange (PT_SECTOR_PROX=0 keeps it replicated)
    static const bool env = [] {
        const char* e = getenv("PT_SECTOR_PROX");
        return !(e && e[0] == '0');
    }();
    if (env && world > 1 && P->Z == 1 && P->Hg == P->H && s->d.prox_kind == 1 &&
        api.send && api.recv && api.group_start &&
        api.group_end && api.bcast && P->H / world >= pt::kRowGhost) {
        s->sr0 = sector_row(P->H, rank, world);
        s->sHl = sector_row(P->H, rank + 1, world) - s->sr0;
        PT_CHECK_CUDA(cudaMalloc(&s->rows_work,
                                 (size_t)pt::fgp2d_slab_floats(s->sHl, P->W) * sizeof(float)));
        s->rhalo.rank = rank;
        s->rhalo.world = world;
        s->rhalo.ctx = s;
        s->rhalo.exchange = nccl_rows_halo;
        s->sector_rows = true;
    }
    return build_selections(s);
}

int attach_zslab(pt_session* s, const NcclApi& api, nccl_comm comm, int rank, int world,
                 int32_t z_offset, int32_t z_total)
{
    pt_plan* P = s->plan;
    if (z_offset < 0 || z_total < 2 || z_offset + P->Z > z_total) {
        pt::set_error("slab [%d, %d) outside a volume of %d planes", z_offset, z_offset + P->Z, z_total);
        return PT_EINVAL;
    }
    if (!api.send || !api.recv || !api.group_start || !api.group_end) {
        pt::set_error("libnccl lacks ncclSend/ncclRecv");
        return PT_ENCCL;
    }
    if (s->d.prox_kind == 1) {
        PT_CHECK_CUDA(cudaMalloc(&s->fgp3_work,
                                 (size_t)pt::fgp3d_slab_floats(P->Z, P->H, P->W) * sizeof(float)));
        if (!s->dw) PT_CHECK_CUDA(cudaMalloc(&s->dw_slab, s->n * sizeof(float)));
    }
    s->nccl = api;
    s->comm = comm;
    s->rank = rank;
    s->world = world;
    s->zslab = true;
    s->z0 = z_offset;
    s->Zg = z_total;
    s->halo.rank = rank;
    s->halo.world = world;
    s->halo.ctx = s;
    s->halo.exchange = nccl_halo;
    return build_selections(s);
}

int attach_rows(pt_session* s, const NcclApi& api, nccl_comm comm, int rank, int world,
                int32_t row_offset, int32_t rows_total)
{
    pt_plan* P = s->plan;
    if (P->Z != 1 || P->row0 != row_offset || P->Hg != rows_total) {
        pt::set_error("the session's plan is not the row slab [%d, %d) of %d rows", row_offset,
                      row_offset + P->H, rows_total);
        return PT_EINVAL;
    }
    if (!api.send || !api.recv || !api.group_start || !api.group_end) {
        pt::set_error("libnccl lacks ncclSend/ncclRecv");
        return PT_ENCCL;
    }
    if (s->d.prox_kind == 1 && world > 1 && P->H < pt::kRowGhost) {
        pt::set_error("a row slab needs at least %d rows for the TV prox", pt::kRowGhost);
        return PT_EINVAL;
    }
    PT_CHECK_CUDA(cudaMalloc(&s->y64, (size_t)P->A * P->Z * P->B * sizeof(double)));
    if (s->d.prox_kind == 1)
        PT_CHECK_CUDA(cudaMalloc(&s->rows_work,
                                 (size_t)pt::fgp2d_slab_floats(P->H, P->W) * sizeof(float)));
    s->nccl = api;
    s->comm = comm;
    s->rank = rank;
    s->world = world;
    s->rows = true;
    s->rhalo.rank = rank;
    s->rhalo.world = world;
    s->rhalo.ctx = s;
    s->rhalo.exchange = nccl_rows_halo;
    return build_selections(s);
}

}  // namespace

int pt_session_override_rank(pt_session* s, int32_t rank, int32_t world)
{
    if (!s || world < 1 || rank < 0 || rank >= world) { pt::set_error("bad argument"); return PT_EINVAL; }
    if (!s->comm) { pt::set_error("session is not attached"); return PT_EINVAL; }
    s->rank = rank;
    s->world = world;
    return build_selections(s);
}

int pt_session_attach_comm_rows(pt_session* s, pt_comm* c, int32_t row_offset, int32_t rows_total)
{
    if (!s || !c) { pt::set_error("null argument"); return PT_EINVAL; }
    if (s->comm) { pt::set_error("session already attached"); return PT_EINVAL; }
    return attach_rows(s, c->api, c->comm, c->rank, c->world, row_offset, rows_total);
}

int pt_session_attach_comm(pt_session* s, pt_comm* c)
{
    if (!s || !c) { pt::set_error("null argument"); return PT_EINVAL; }
    if (s->comm) { pt::set_error("session already attached"); return PT_EINVAL; }
    return attach_sector(s, c->api, c->comm, c->rank, c->world);
}

int pt_session_attach_comm_zslab(pt_session* s, pt_comm* c, int32_t z_offset, int32_t z_total)
{
    if (!s || !c) { pt::set_error("null argument"); return PT_EINVAL; }
    if (s->comm) { pt::set_error("session already attached"); return PT_EINVAL; }
    return attach_zslab(s, c->api, c->comm, c->rank, c->world, z_offset, z_total);
}

int pt_session_attach_nccl_zslab(pt_session* s, const char* nccl_path, const uint8_t* host_id128,
                                 int32_t rank, int32_t world, int32_t z_offset, int32_t z_total)
{
    if (!s || !host_id128 || world < 1 || rank < 0 || rank >= world) { pt::set_error("bad argument"); return PT_EINVAL; }
    if (s->comm) { pt::set_error("session already attached"); return PT_EINVAL; }
    pt_comm* c = nullptr;
    int rc = pt_nccl_comm_create(nccl_path, host_id128, rank, world, &c);
    if (rc) return rc;
    rc = attach_zslab(s, c->api, c->comm, rank, world, z_offset, z_total);
    if (rc) {
        pt_nccl_comm_destroy(c);
        s->comm = nullptr;
        s->zslab = false;
        return rc;
    }
    s->owns_comm = true;
    delete c;  // the session owns the communicator now
    return PT_OK;
}

int pt_session_attach_nccl(pt_session* s, const char* nccl_path, const uint8_t* host_id128,
                           int32_t rank, int32_t world)
{
    if (!s || !host_id128 || world < 1 || rank < 0 || rank >= world) { pt::set_error("bad argument"); return PT_EINVAL; }
    if (s->comm) { pt::set_error("session already attached"); return PT_EINVAL; }
    // world == 1 is accepted: a one-rank communicator exercises the whole
    // sharded data path (partial gradient -> ncclAllReduce -> epilogue)
    pt_comm* c = nullptr;
    int rc = pt_nccl_comm_create(nccl_path, host_id128, rank, world, &c);
    if (rc) return rc;
    rc = attach_sector(s, c->api, c->comm, rank, world);
    if (rc) {
        pt_nccl_comm_destroy(c);
        s->comm = nullptr;
        return rc;
    }
    s->owns_comm = true;
    delete c;  // the session owns the communicator now
    return PT_OK;
}

}  // extern "C"
