/*
 * proxtomo_b200.h -- C ABI of the B200-native ProxSkip-VR CT hot path.
 *
 * The reference (`proxtomo`, arxiv/paper_2602_09527) is pure Python; its seam
 * for this path is a duck-typed projector object plus plain functions.  Each
 * entry point below replaces one reference call; the reference symbol it
 * stands in for is cited as pkg/src/proxtomo/<file>:<lines>.
 *
 * Conventions
 *  - Every array argument is a caller-owned DEVICE pointer (float32, row-major,
 *    contiguous) unless its name starts with `host_`.
 *  - Images are (n_slices, height, width); n_slices == 1 is the 2D case.
 *    Sinograms are (n_angles, n_slices, n_bins) (angle-major, so a subset is a
 *    set of whole angle blocks); a selection's output is (n_sel, n_slices, n_bins).
 *  - Every compute call is stream-ordered on `stream` (a cudaStream_t passed
 *    as void*), performs no allocation and no host synchronisation unless
 *    documented ("syncs").
 *  - Return value: PT_OK (0) or a negative PT_E* code; pt_last_error() gives
 *    the message of the calling thread's last failure.  PT_EINVAL maps to the
 *    reference's ValueError, PT_ECUDA / PT_ENCCL to RuntimeError.
 *  - A plan is immutable after creation (selections are added under a lock)
 *    and may be shared by threads using distinct sessions / streams.
 */
#ifndef PROXTOMO_B200_H
#define PROXTOMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PT_OK 0
#define PT_EINVAL -1
#define PT_ECUDA -2
#define PT_EUNSUPPORTED -3
#define PT_ENCCL -4

typedef struct pt_plan pt_plan;
typedef struct pt_selection pt_selection;
typedef struct pt_session pt_session;

/* Scan geometry + image grid.  Replaces ParallelGeometry
 * (pkg/src/proxtomo/geometry.py:9-47) bound to a grid by Projector
 * (pkg/src/proxtomo/projector.py:143-153).  `host_angles` are radians,
 * validated like the reference (strictly increasing, in [0, pi)). */
typedef struct {
    int32_t height, width;   /* image grid (H, W) */
    int32_t n_slices;        /* >= 1; > 1 = slice-stacked 3D (rotation about z) */
    int32_t n_angles, n_bins;
    double bin_spacing, pixel_size;
    const double* host_angles;
    /* Row slab (multi-GPU rows decomposition): the plan's grid is rows
     * [row_offset, row_offset + height) of a rows_total-row image; the
     * projector's A and A^T are the whole image's restricted to those rows
     * (forward partial sums add up over the slabs).  rows_total = 0: the
     * grid is the whole image. */
    int32_t row_offset, rows_total;
} pt_geometry_desc;

const char* pt_last_error(void);
const char* pt_version(void);
/* Process-wide number of kernels this library has launched (evidence that
 * the native path, not a fallback, ran). */
int64_t pt_launch_count(void);
/* sizeof(pt_geometry_desc): a binding built from its own copy of the struct
 * (ctypes, cffi, cgo) asserts this at load time so a layout change cannot
 * make pt_plan_create read past the caller's struct. */
int64_t pt_geometry_desc_size(void);

/* Plan lifecycle: uploads the per-angle Joseph tables (computed on the host
 * in float64 from the reference's expressions, projector.py:26-61). */
int pt_plan_create(const pt_geometry_desc* desc, pt_plan** out);
int pt_plan_destroy(pt_plan* plan);

/* An angle selection (a subset, projector.py:86-97 `pair(subset)`); NULL
 * host_idx with n == -1 means all angles in order.  Index validation as
 * projector.py:105-111.  Selections live as long as the plan. */
int pt_selection_create(pt_plan* plan, const int32_t* host_idx, int32_t n, pt_selection** out);
int32_t pt_selection_size(const pt_selection* sel);
/* Sum over the selection of the number of nonzero Joseph weights (the
 * reference's CSR nnz of A_S, projector.py:55-60), host-side count. */
int64_t pt_selection_nnz(pt_plan* plan, const pt_selection* sel);

/* y = A_S (x - x2) [- b_S].  Replaces forward_project (projector.py:114-126)
 * and the residual of _subset_gradient (estimators.py:29-31).
 * x2 (may be NULL) is subtracted before projection (SVRG: A_i(x - x_snap));
 * data (may be NULL) is the FULL sinogram (n_angles, n_slices, n_bins) whose
 * selected rows are subtracted; sumsq (may be NULL, device double[1]) receives
 * sum(y^2) (objective, solvers.py:271-277).  Uses the plan's workspace:
 * standalone calls on one plan must be serialised on one stream. */
int pt_forward(pt_plan* plan, const pt_selection* sel, const float* x, const float* x2,
               const float* data, float* y, double* sumsq, void* stream);

/* x_out = alpha * A_S^T y (+ beta * x_out when accumulate != 0).  Replaces
 * back_project (projector.py:129-140); a per-pixel gather, no atomics,
 * deterministic. */
int pt_adjoint(pt_plan* plan, const pt_selection* sel, const float* y, float* x_out,
               float alpha, int32_t accumulate, void* stream);

/* Estimator kinds (estimators.py:24). */
#define PT_EST_FULL 0
#define PT_EST_SGD 1
#define PT_EST_SAGA 2
#define PT_EST_SVRG 3
#define PT_EST_LSVRG 4
/* Session-only kinds (not an estimator of the reference, a solver of it):
 * FISTA (solvers.py:367-392) -- per step the full gradient at the momentum
 * point y, x+ = prox_gamma(y - gamma grad f(y)), y = x+ + beta_k (x+ - x) with
 * t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2, beta_k = (t_k - 1) / t_{k+1}, t_1 = 1
 * (the t sequence is kept in float64 on the host side of the session).
 * ISTA (:339-364) is PT_EST_FULL with skip_probability 1 (hcoef = 0). */
#define PT_EST_FISTA 5

/* Fused adjoint + estimator + ProxSkip gradient half-step, one pass:
 *   g    = A_S^T r                              (estimators.py:32)
 *   est  = g | N g | N g + (S - N T_i) | N g + G (full/sgd/saga/svrg)
 *          (estimators.py:55,92,146); SAGA also S <- (S - T_i) + g, T_i <- g
 *          (estimators.py:93-94)
 *   base = x - gamma est; x_hat = base + gamma h (solvers.py:236-237)
 *   theta == 0: x_out = x_hat                   (solvers.py:246)
 *   theta == 1: v_out = base + hcoef h, xhat_out = x_hat, hcoef = gamma - gamma/p
 *               (solvers.py:242)
 * A non-finite x_out sets *bad_iter = min(*bad_iter, iteration) (device int64;
 * DivergenceError, solvers.py:247-248).  For SVRG, r must be A_i(x - x_snap)
 * (b cancels) and aux0 = full_grad; for SAGA aux0 = table_i, aux1 = sum. */
typedef struct {
    int32_t estimator;
    int32_t theta;
    float n_scale;       /* N */
    float gamma;
    float hcoef;
    int64_t iteration;
    const float* x;
    const float* h;
    float* aux0;
    float* aux1;
    float* x_out;
    float* v_out;
    float* xhat_out;
    int64_t* bad_iter;
} pt_step_epilogue;

int pt_adjoint_step(pt_plan* plan, const pt_selection* sel, const float* r,
                    const pt_step_epilogue* ep, void* stream);
/* The same epilogue applied to an already-reduced gradient g (multi-GPU path:
 * partial A^T r per angle sector -> allreduce -> this). */
int pt_step_epilogue_apply(pt_plan* plan, const float* g, const pt_step_epilogue* ep,
                           void* stream);

/* FGP TV prox (regularizers.py:90-133), temporally blocked.  v: prox input;
 * lam = tau * alpha; p, q (and w in 3D) are the warm duals in/out (zeros =
 * cold start; the caller applies the reference's reuse rule, :102-106);
 * x_out = max(v - lam D^T(p,q), 0 if nonneg).  When h != NULL the ProxSkip
 * control-variate update h += p_over_gamma (x_out - xhat) is fused into the
 * last launch (solvers.py:249-250) and non-finite x_out raises *bad_iter.
 * `work` is a device buffer of pt_fgp_workspace_floats() floats. */
int64_t pt_fgp_workspace_floats(pt_plan* plan);
int pt_tv_prox(pt_plan* plan, const float* v, double lam, int32_t inner_iterations,
               int32_t nonneg, float* p, float* q, float* w, float* x_out, const float* xhat,
               float* h, float p_over_gamma, int64_t iteration, int64_t* bad_iter, float* work,
               void* stream);

/* Test hook of the multi-GPU row decomposition: the 2D TV prox of the
 * whole image run as `slabs` row slabs on this device (ghost-row copies
 * standing in for the NCCL halo exchange).  Arguments as
 * pt_tv_prox on whole-image arrays; the result equals pt_tv_prox bitwise. */
int pt_tv_prox_emulate_rows(pt_plan* plan, int32_t slabs, const float* v, double lam,
                            int32_t inner_iterations, int32_t nonneg, float* p, float* q,
                            float* x_out, void* stream);

/* Reductions into device doubles (deterministic: fixed grid and combine
 * order, float64 accumulation).  `out` must hold PT_RED_DOUBLES doubles:
 * out[0] (and out[1] for pt_diff_norms) is the result, the rest scratch. */
#define PT_RED_DOUBLES 1025
int pt_dot(const float* a, const float* b, int64_t n, double* out, void* stream);
/* isotropic TV, forward differences (regularizers.py:79-82; 3D adds z) */
int pt_tv_value(pt_plan* plan, const float* x, double* out, void* stream);
/* out[0] = sum((x - ref)^2), out[1] = sum(ref^2)   (metrics.py:19-27) */
int pt_diff_norms(const float* x, const float* ref, int64_t n, double* out, void* stream);

/* Squared operator norm by the reference's Rayleigh power method
 * (projector.py:170-197); v0 is the host-drawn start vector (device copy,
 * overwritten).  Syncs; returns the estimate in *host_out. */
int pt_operator_norm_sq(pt_plan* plan, float* v0, int32_t iterations, double* host_out,
                        void* stream);

/* Diagonally preconditioned PDHG reference solver, elementwise steps
 * (solvers.py:395-455; the projector calls are pt_forward with the data
 * subtraction and pt_adjoint).  Images are (n_slices, height, width) stacks
 * of independent 2D planes (the reference is 2D: n_slices = 1).
 *   dual_sino: y = (y + sigma_a * resid) / (1 + sigma_a)                (:434)
 *   dual_tv:   (zv, zh) = clip to |.| <= alpha of (zv, zh) + sigma_d D xbar (:436-442)
 *   primal:    x' = x - tau (ascent + D^T(zv, zh)) [max(., 0) if nonneg];
 *              xbar = 2 x' - x; x = x'; zv == NULL skips the TV term;
 *              non-finite x' lowers *bad_iter to `iteration`        (:443-451) */
int pt_pdhg_dual_sino(float* y, const float* resid, const float* sigma_a, int64_t n,
                      void* stream);
int pt_pdhg_dual_tv(const float* xbar, float* zv, float* zh, int32_t n_slices, int32_t height,
                    int32_t width, double sigma_d, double alpha, void* stream);
int pt_pdhg_primal(float* x, float* xbar, const float* ascent, const float* zv, const float* zh,
                   const float* tau, int32_t n_slices, int32_t height, int32_t width,
                   int32_t nonneg, int64_t iteration, int64_t* bad_iter, void* stream);

/* ------------------------------------------------------------------ */
/* Native executor for the ProxSkip loop (solvers.py:159-324).          */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t estimator;       /* PT_EST_* */
    int32_t n_subsets;
    double gamma;
    double skip_probability; /* p */
    int32_t prox_kind;       /* 0 identity, 1 TV (FGP) */
    double tv_alpha;
    int32_t tv_inner;
    int32_t tv_warm_start;
    int32_t tv_nonneg;
} pt_solver_desc;

/* data: full sinogram (device, n_angles x n_slices x n_bins), must outlive the
 * session.  x0 may be NULL (zeros, solvers.py:161). */
int pt_session_create(pt_plan* plan, const pt_solver_desc* desc, const float* data,
                      const float* x0, pt_session** out, void* stream);
/* The same with caller-provided device memory for every session buffer (state,
 * divergence flag, projector workspace): `workspace` of at least
 * pt_session_workspace_bytes() bytes, 256-byte aligned, owned by the caller and
 * kept alive until pt_session_destroy (e.g. from a caching allocator, so
 * repeated solves do not cudaMalloc). */
int64_t pt_session_workspace_bytes(pt_plan* plan, const pt_solver_desc* desc);
int pt_session_create_in(pt_plan* plan, const pt_solver_desc* desc, const float* data,
                         const float* x0, void* workspace, int64_t workspace_bytes,
                         pt_session** out, void* stream);
int pt_session_destroy(pt_session* s);
/* SVRG/LSVRG initial snapshot + full gradient (estimators.py:117-123). */
int pt_session_init(pt_session* s, void* stream);
/* Enqueue n_steps iterations k0 .. k0+n_steps-1 of proxskip_step
 * (solvers.py:230-254).  host_subset[j]: drawn subset index (ignored for
 * full); host_theta[j]: Bernoulli(p) outcome; host_refresh[j]: SVRG snapshot
 * refresh before step j (estimators.py:149-162).  No host sync. */
int pt_session_run(pt_session* s, int32_t n_steps, const int32_t* host_subset,
                   const uint8_t* host_theta, const uint8_t* host_refresh, int64_t k0,
                   void* stream);
/* The same for a whole run planned on the host: after step host_marks[m]
 * (cumulative, ascending) the cudaEvent_t events[m] is recorded on `stream`
 * (the log rows' device times, solvers.py:304-322), so a run whose rows need
 * no metric is one call.  No host sync. */
int pt_session_run_marked(pt_session* s, int32_t n_steps, const int32_t* host_subset,
                          const uint8_t* host_theta, const uint8_t* host_refresh, int64_t k0,
                          int32_t n_marks, const int32_t* host_marks, void* const* events,
                          void* stream);
/* Device pointers of the live state (valid until the next run call). */
float* pt_session_x(pt_session* s);
float* pt_session_h(pt_session* s);
float* pt_session_buffer(pt_session* s, int32_t which); /* 0 snapshot 1 full_grad 2 saga sum 3 saga table 4 dual p 5 dual q */
int64_t* pt_session_bad_iter(pt_session* s);            /* device int64, INT64_MAX = finite */

/* Per-kernel-category device time inside pt_session_run / _init (CUDA events
 * on the session stream around each launch; off by default). */
#define PT_PROF_FWD_BAND 0   /* forward band-partial kernel (per-step subset) */
#define PT_PROF_FWD_REDUCE 1 /* forward band reduction (+ residual)           */
#define PT_PROF_GATHER 2     /* fused gather + estimator + ProxSkip epilogue  */
#define PT_PROF_FGP 3        /* one TV prox call (all its launches)           */
#define PT_PROF_SNAPSHOT 4   /* SVRG snapshot full gradient (fwd + adj)       */
#define PT_PROF_OTHER 5      /* copies, identity prox, allreduce              */
/* the snapshot's own launches (also inside PT_PROF_SNAPSHOT's time) */
#define PT_PROF_SNAP_FWD_BAND 6
#define PT_PROF_SNAP_FWD_REDUCE 7
#define PT_PROF_SNAP_GATHER 8
#define PT_PROF_N 9
int pt_session_set_profiling(pt_session* s, int32_t on);
/* Syncs the session stream; returns accumulated ms and call counts per
 * category since the last collection, then resets them. */
int pt_session_profile(pt_session* s, double* host_ms, int64_t* host_calls);

/* Multi-GPU (angle sectors).  The NCCL library is dlopen'ed from `nccl_path`
 * (the torch-bundled libnccl.so.2), so this .so has no link-time NCCL.
 * unique_id: 128 bytes from pt_nccl_unique_id on rank 0, broadcast by the
 * caller.  After attach, the session's per-step subset gradients cover only
 * angles [rank*A/world, (rank+1)*A/world) and are summed by ncclAllReduce on
 * the session stream before the epilogue (world == 1 runs that path on a
 * one-rank communicator). */
int pt_nccl_unique_id(const char* nccl_path, uint8_t* host_out128);
/* A process-level communicator shared by several sessions (one
 * ncclCommInitRank per process group instead of one per solve); destroy it
 * after the last session that uses it. */
typedef struct pt_comm pt_comm;
int pt_nccl_comm_create(const char* nccl_path, const uint8_t* host_id128, int32_t rank,
                        int32_t world, pt_comm** out);
int pt_nccl_comm_destroy(pt_comm* comm);
/* attach a session to a shared communicator: angle sectors / z-slabs */
int pt_session_attach_comm(pt_session* s, pt_comm* comm);
int pt_session_attach_comm_zslab(pt_session* s, pt_comm* comm, int32_t z_offset,
                                 int32_t z_total);
/* Image-rows decomposition of a 2D problem: the session's plan is the row
 * slab [row_offset, row_offset + height) of a rows_total-row image
 * (pt_geometry_desc.row_offset / rows_total), its state the slab's rows.
 * Every forward's partial line integrals are summed over the ranks in
 * float64 (ncclAllReduce, 8 |S| B bytes); the gather, step and TV prox touch
 * only the own rows (the prox exchanges 9 ghost rows with ranks -+ 1 per
 * launch, ncclSend / ncclRecv).  Needs >= 9 rows per rank. */
int pt_session_attach_comm_rows(pt_session* s, pt_comm* comm, int32_t row_offset,
                                int32_t rows_total);
int pt_session_attach_nccl(pt_session* s, const char* nccl_path, const uint8_t* host_id128,
                           int32_t rank, int32_t world);
/* Test hook: make an attached session believe it is rank `rank` of `world`
 * while its communicator keeps its real size (a one-rank communicator then
 * exercises the per-rank offsets of the slab layouts, e.g. the snapshot
 * residual's angle indexing in rows mode, on one GPU).  Only for runs that
 * exchange no halos (no TV prox).  Call before pt_session_init. */
int pt_session_override_rank(pt_session* s, int32_t rank, int32_t world);
/* Test hook: run the angle-sector decomposition of `world` ranks on this one
 * device (each sector's partial A_i^T r computed separately and summed, which
 * is exactly what ncclAllReduce sums across real ranks).  Call before run. */
int pt_session_emulate_sectors(pt_session* s, int32_t world);

/* z-slab decomposition of a slice-stacked 3D volume: the
 * session's plan holds this rank's planes [z_offset, z_offset + Z) of a
 * z_total-plane volume and `data` its sinogram rows (A, Z, B).  The projector,
 * gradients and snapshot are slab-local (rays never cross slices); the 3D TV
 * prox exchanges one boundary plane of the duals per inner iteration (and of
 * its input once per call) with ranks -+ 1 by ncclSend/ncclRecv on the
 * session stream.  Ranks must hold consecutive slabs in rank order. */
int pt_session_attach_nccl_zslab(pt_session* s, const char* nccl_path, const uint8_t* host_id128,
                                 int32_t rank, int32_t world, int32_t z_offset, int32_t z_total);
/* Test hook: run the 3D TV prox as `slabs` virtual z-slabs of this volume on
 * one device (each slab sees its neighbours only through its ghost planes,
 * filled by device copies).  Call before run. */
int pt_session_emulate_zslabs(pt_session* s, int32_t slabs);

#ifdef __cplusplus
}
#endif
#endif /* PROXTOMO_B200_H */
