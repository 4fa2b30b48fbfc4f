/*
 * whb200 — B200-native (sm_100a) WaveHoltz explicit iteration, C ABI.
 *
 * This is the drop-in boundary under the reference package's Python
 * solve/iterate surface (waveholtz 0.1.0).  The reference has no FFI of its
 * own: its boundary is the Python function surface resolved by module-level
 * name lookup (driver.py:38 imports wave_solve_filtered by name), so each
 * entry point below states which reference function (file:line under
 * /root/reference/pkg/src/waveholtz) it replaces.  The Python host package
 * paper_2504_03074_b200 binds these with ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or CUDA types in signatures.
 *  - Every call returns 0 on success or a negative WHB_E* code; the message
 *    of the last failure on the calling thread is whb_last_error().
 *  - Host pointers are borrowed for the duration of the call only.
 *  - Fields are float64, C-contiguous in grid.shape with 'ij' indexing
 *    (grid.py:109-112); Dirichlet boundary points are exactly 0.
 *  - All per-step scalars (cos(wt*(n*dt)), (cos-alpha/2)*sigma, dt^2/2, dt^2,
 *    (2/Tbar)*dt, stencil coefficients (1,-2,1)/dx^2, c^2) are computed by the
 *    caller exactly as the reference computes them (timestep.py:134-145,
 *    250-301; grid.py:302-306, 366) so device libm never enters the results.
 *    The kernels are compiled without FMA contraction, so iterates are
 *    bitwise identical to the reference.
 *  - A context lives on one device and owns all of its device buffers and
 *    one CUDA stream; calls on one context must come from one host thread.
 */
#ifndef WHB200_H
#define WHB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WHB_ABI_VERSION 2

/* Ghost planes allocated on each side of a context's owned axis-0 planes. */
#define WHB_GHOST_PLANES 3

enum whb_status {
    WHB_OK = 0,
    WHB_E_ARG = -1,      /* invalid argument (Python: ValueError)             */
    WHB_E_CUDA = -2,     /* CUDA runtime failure (Python: RuntimeError)       */
    WHB_E_NOMEM = -3,    /* device/host allocation failed (MemoryError)       */
    WHB_E_STATE = -4,    /* call out of order, e.g. no schedule set           */
    WHB_E_NODEV = -5     /* no CUDA device visible                            */
};

/* Field slots of a batch member (per member unless shared). */
enum whb_field {
    WHB_V = 0,    /* iterate v (W^0 of a solve; FPI updates it in place)      */
    WHB_F = 1,    /* forcing f(x) (shared by all members if shared_forcing)   */
    /* Time levels L >= 1 live in a ring of nring buffers, level L in slot L mod nring
     * (whb_plan reports the kernel family; nring = 6 for plans with 4-step passes, 4 otherwise).
     * A pass of T steps reads levels s, s-1 and writes s+T-1, s+T; nring >= T + 2 keeps the
     * written slots disjoint from the read ones.  WA..WD name ring slots 1, 2, 3 and 0; slots
     * 4 and 5 of a 6-slot ring are internal. */
    WHB_WA = 2,   /* ring slot 1                                               */
    WHB_WB = 3,   /* ring slot 2                                               */
    WHB_ACC = 4,  /* running filter sum                                        */
    WHB_OUT = 5,  /* output of a plain/matvec solve                            */
    WHB_WC = 6,   /* ring slot 3                                               */
    WHB_WD = 7    /* ring slot 0                                               */
};

/* What the last step of a filtered solve writes (timestep.py:300-301, driver.py:222-225, 256-262). */
enum whb_out_mode {
    WHB_OUT_PLAIN = 0, /* OUT = (2/Tbar)dt*acc                    — wave_solve_filtered  */
    WHB_OUT_FPI = 1,   /* V <- (2/Tbar)dt*acc ; resid += (V_new - V_old)^2 — _iterate    */
    WHB_OUT_AV = 2     /* OUT = V - (2/Tbar)dt*acc  (V = x, f ignored)     — A x = x - W(x,0) */
};

typedef struct whb_ctx whb_ctx;

int whb_abi_version(void);
const char *whb_last_error(void);
int whb_device_count(int *count);

/*
 * Create a context for `nbatch` independent problems on one grid.
 *   ndim in {1,2,3}; shape[ndim] = grid.shape (stored points, grid.py:85-94).
 *   [plane_begin, plane_end): the global axis-0 planes this context owns
 *   (slab decomposition); pass 0, shape[0] for the whole grid.  ndim==1
 *   must own the whole grid.
 *   shared_forcing != 0: one f for all members (batched frequencies, cfg 5).
 * Replaces: CartesianGrid/GridField storage (grid.py:50-291) + WaveState
 * (timestep.py:111-129) buffers.
 */
int whb_create(whb_ctx **out, int device, int ndim, const int64_t *shape, int64_t plane_begin,
               int64_t plane_end, int nbatch, int shared_forcing);
int whb_destroy(whb_ctx *ctx);

/* c^2 * Laplacian_h coefficients per axis: clo[a] = 1/dx_a^2, cmid[a] = -2/dx_a^2
 * (stencil_coefficients, grid.py:302-306) and c2 = c**2 (grid.py:366).
 * Replaces DiscreteOperator (grid.py:309-368), order p = 2, all-Dirichlet. */
int whb_set_operator(whb_ctx *ctx, const double *clo, const double *cmid, double c2);

/* General operator: order p in {2, 4} and per-axis boundary
 * conditions — periodic[a] != 0: wrap-around, else homogeneous Dirichlet closed by
 * odd reflection (grid.py:371-392).  taps[a*(p+1) + q] = stencil_coefficients(p, dx_a)[q]
 * (grid.py:296-306), c2 = c**2.  Whole-grid contexts only.  Runs a one-step-per-pass
 * kernel (the temporal-blocked kernels implement p = 2, all-Dirichlet). */
int whb_set_operator_general(whb_ctx *ctx, int order, const int *periodic, const double *taps, double c2);

/* Per-member time schedule of one filtered solve (n_total = N_p*N_t steps):
 *   cos_f[n_total]   cos(wt*(n*dt)) forcing factor of step n (entry 0 unused)
 *   acc_c[n_total+1] (cos(wt*(n*dt)) - alpha/2)*sigma_n filter weights
 * Replaces the scalar part of wave_solve_filtered/step_explicit
 * (timestep.py:134-145, 271-300) with correct_explicit (timestep.py:78-97). */
int whb_set_schedule(whb_ctx *ctx, int member, int n_total, double half_dt2, double dt2,
                     const double *cos_f, const double *acc_c, double out_scale);

/* Field I/O.  `host` holds the owned planes [plane_begin, plane_end) of the
 * field, C-contiguous.  Upload re-zeroes Dirichlet boundary points
 * (GridField.set_values, grid.py:218-227).  member is ignored for a shared f. */
int whb_upload(whb_ctx *ctx, int field, int member, const double *host);
int whb_download(whb_ctx *ctx, int field, int member, double *host);
/* The same with a strided host view (e.g. the interior of a ghost-padded GridField buffer,
 * grid.py:185-216): element strides between storage planes and between rows, the last axis
 * contiguous; one 3D copy, no host-side packing. */
int whb_upload_strided(whb_ctx *ctx, int field, int member, const double *host, int64_t plane_stride,
                       int64_t row_stride);
int whb_download_strided(whb_ctx *ctx, int field, int member, double *host, int64_t plane_stride,
                         int64_t row_stride);
int whb_zero(whb_ctx *ctx, int field, int member);

/* One filtered solve W(v, f) for every member, device resident
 * (wave_solve_filtered, timestep.py:250-301, explicit branch).
 *   zero_forcing != 0: f treated as 0 (waveholtz_operator, driver.py:254-258).
 *   resid_sq (host, nbatch entries, may be NULL): WHB_OUT_FPI only,
 *   sum over owned points of (v_new - v_old)^2 (driver.py:225 before sqrt). */
int whb_filtered_solve(whb_ctx *ctx, int out_mode, int zero_forcing, double *resid_sq);

/* `iters` fixed-point passes v <- W(v, f) for all members (driver.py:211-230).
 * resid_sq_out[iters*nbatch] (host, may be NULL) receives sum (v_{k+1}-v_k)^2
 * per iteration and member (the caller divides by N and takes sqrt).
 * tol_sq >= 0: stop after the first iteration whose resid_sq <= tol_sq for
 * every member (checked on the host each iteration); tol_sq < 0: run all
 * iterations with no host synchronisation in between.
 * iters_done (may be NULL) receives the number of passes run. */
int whb_fpi(whb_ctx *ctx, int iters, double tol_sq, double *resid_sq_out, int *iters_done);

/* whb_fpi with the reference's own stopping test (driver.py:225-230): stop after
 * the first iteration with sqrt(resid_sq) / root_n <= tol for every member
 * (IEEE sqrt and division, so the decision is the host loop's bit for bit;
 * root_n = sqrt(N) as the caller computes it, > 0; tol < 0: never stop early).
 * Cluster-resident grids (whb_plan kernel 4, one member) take the test inside
 * the kernel: the whole tol-driven fpi_solve is one launch. */
int whb_fpi_scaled(whb_ctx *ctx, int iters, double tol, double root_n, double *resid_sq_out, int *iters_done);

/* End-to-end single-member pass with host buffers (member 0): copy v_host
 * H2D, v <- W(v, f), copy v D2H into v_out_host, resid_sq as in whb_fpi.
 * The drop-in for one call of wave_solve_filtered inside _iterate
 * (driver.py:222-225) with host GridFields. */
int whb_iterate_host(whb_ctx *ctx, const double *v_host, double *v_out_host, double *resid_sq);

/* wave_solve_filtered (timestep.py:250-301) with host fields on both sides, member 0: v_host ->
 * device, one filtered solve in `out_mode` (WHB_OUT_PLAIN: W(v, f); WHB_OUT_AV: v - W(v, 0), the
 * mat-vec of driver.py:262-267; WHB_OUT_FPI: as whb_iterate_host), result -> out_host.  Both host
 * fields are strided views as in whb_upload_strided (element strides of planes and rows; a
 * reference GridField's ghost-padded buffer is such a view).  v_host is not modified unless it
 * aliases out_host.  On whole-grid 3D problems that run the three-step plan the transfers are
 * hidden behind the passes: v moves in bands of rows on copy streams while the (pass, band)
 * launches follow diagonal by diagonal (same arithmetic per point as the whole-grid launches:
 * the result is bitwise the same); otherwise upload, solve, download in sequence. */
int whb_solve_host(whb_ctx *ctx, const double *v_host, int64_t v_plane_stride, int64_t v_row_stride,
                   double *out_host, int64_t out_plane_stride, int64_t out_row_stride, int out_mode,
                   int zero_forcing, double *resid_sq);

/* ---- Krylov vectors (gmres_solve, linalg.py:102-183; member 0 only) ------
 * Vector ids >= 0 name full-grid device vectors with the field layout.
 * Slots: ids WHB_V..WHB_WD alias the member-0 fields; ids >= 8 are extra
 * vectors reserved with whb_vec_reserve.  Reductions are deterministic
 * (fixed-order tree), over owned points. */
int whb_vec_reserve(whb_ctx *ctx, int count, int *first_id);
int whb_vec_upload(whb_ctx *ctx, int id, const double *host);
int whb_vec_download(whb_ctx *ctx, int id, double *host);
int whb_vec_dot(whb_ctx *ctx, int x, int y, double *out);                    /* np.vdot, linalg.py:145 */
int whb_vec_axpy(whb_ctx *ctx, double a, int x, int y);                       /* y += a*x, linalg.py:146 */
int whb_vec_scale_into(whb_ctx *ctx, double a, int x, int y);                 /* y = x*a  */
int whb_vec_div_into(whb_ctx *ctx, int x, double d, int y);                   /* y = x/d, linalg.py:150 */
int whb_vec_lincomb(whb_ctx *ctx, int y, int first, int count, const double *coef); /* y += Q[:,first:first+count]@coef, linalg.py:174 */
int whb_vec_sub_into(whb_ctx *ctx, int x, int y, int z);                      /* z = x - y */
int whb_vec_copy(whb_ctx *ctx, int x, int y);                                 /* y = x */
/* Modified Gram-Schmidt against basis vectors q_first .. q_first+count-1 on the device
 * (linalg.py:143-150): for j: h[j] = q_j.w; w -= h[j] q_j; then h[count] = w.w and, when
 * q_next >= 0 and h[count] > 0, q_next = w / sqrt(h[count]).  h_out[count+1] (host) receives
 * the coefficients after one synchronisation (the per-dot host round trips of the vector
 * calls above disappear). */
int whb_vec_mgs(whb_ctx *ctx, int w, int q_first, int count, int q_next, double *h_out);
/* y = c^2 * L_h x at interior points, boundary 0 (DiscreteOperator.apply_values,
 * grid.py:346-368; p = 2, Dirichlet). */
int whb_apply_operator(whb_ctx *ctx, int x, int y);
/* y = x - W(x, 0)  (waveholtz_operator.matvec, driver.py:256-262) */
int whb_matvec(whb_ctx *ctx, int x, int y);

/* ---- slab decomposition (multi-GPU) -------------------------------------
 * Step-level control for halo exchange between contexts on different
 * devices.  Step s of a solve advances W^s -> W^{s+1}.  A solve is
 *   whb_solve_begin; for s: whb_step(s, region); ...; whb_solve_end
 * or, with two leapfrog steps per HBM pass (whb_plan steps_per_pass == 2),
 *   whb_solve_begin; for s = 0, 2, ...: whb_pair(s, region); [whb_step(N-1, 0)]; whb_solve_end,
 * and with three (steps_per_pass == 3, n_total > 3; n_total <= 3 runs the two-step schedule)
 *   whb_solve_begin; for s = 0, 3, ... while N - s >= 3: whb_triple(s, region);
 *   [whb_pair(s, 0) if 2 steps remain | whb_step(s, 0) if 1]; whb_solve_end.
 * Before a pass of k steps the ghosts hold k planes of W^s and k - 1 of W^{s-1}, so after a
 * pass the exchange carries what the NEXT pass needs; F is read k - 1 planes deep.
 * whb_step: region 0 = all owned planes, 1 = the first and last owned update
 * planes only (the planes neighbours need), 2 = the remaining interior planes;
 * W^s needs 1 exchanged ghost plane per side.
 * whb_pair (steps s and s+1): region 0 = all, 1 = the two first and two last
 * update planes, 2 = the rest; W^s needs 2 exchanged ghost planes per side,
 * W^{s-1} and F one (F is static: exchange it once after upload); the last
 * pass of a solve (s + 2 == n_total) must be region 0.
 * Local plane indices: [0, G) low ghosts, [G, G + nloc) owned,
 * [G + nloc, 2G + nloc) high ghosts, G = WHB_GHOST_PLANES (whb_ghost_planes).
 * whb_level_plane_ptr returns the device address of local plane `plane` of
 * the buffer that holds time level `level` of member 0 (level 0 = V);
 * consecutive planes are contiguous (plane_elems apart). */
int whb_solve_begin(whb_ctx *ctx, int out_mode, int zero_forcing);
int whb_step(whb_ctx *ctx, int s, int region);
int whb_pair(whb_ctx *ctx, int s, int region);
/* Three-step pass (s, s+1, s+2) of a context whose plan runs the three-step kernel (whb_plan:
 * 3 steps per pass), with the same regions as whb_pair: 0 = every update plane, 1 = the three
 * first and three last update planes (W^{s+3} there feeds the neighbours' 3 ghost planes, W^{s+2}
 * their 2), 2 = the rest.  Not for a pass that is both the first and the last (N_t = 3). */
int whb_triple(whb_ctx *ctx, int s, int region);
int whb_solve_end(whb_ctx *ctx, double *resid_sq);
int whb_ghost_planes(whb_ctx *ctx, int *ghost);
int whb_level_plane_ptr(whb_ctx *ctx, int level, int64_t plane, uint64_t *dev_ptr, int64_t *plane_elems);
/* the same for a field slot (enum whb_field) of a member, e.g. WHB_F for its ghost exchange */
int whb_field_plane_ptr(whb_ctx *ctx, int field, int member, int64_t plane, uint64_t *dev_ptr,
                        int64_t *plane_elems);
int whb_stream_ptr(whb_ctx *ctx, uint64_t *stream);
int whb_synchronize(whb_ctx *ctx);
/* copy a plane between two contexts (same or peer device), ordered on src's
 * stream then dst's (the single-process multi-shard path). */
int whb_copy_plane(whb_ctx *src, int src_level, int64_t src_plane, whb_ctx *dst, int dst_level,
                   int64_t dst_plane);
/* copy `bytes` between device addresses of two contexts (e.g. several planes from
 * whb_level_plane_ptr / whb_field_plane_ptr), ordered the same way. */
int whb_copy_device(whb_ctx *src, uint64_t src_ptr, whb_ctx *dst, uint64_t dst_ptr, int64_t bytes);

/* ---- implicit trapezoidal stepping ---------------------
 * Vector ids as for whb_vec_*.  The CG iteration (linalg.py:62-99) runs on the
 * host over these calls (paper_2504_03074_b200/implicit.py).
 * whb_imp_apply: y = x - s * c^2 L_h x  (_ImplicitSolver.apply, timestep.py:225-226;
 *   s = 0.5*dt**2; tmp: scratch vector, used by the general operator only).
 * whb_imp_rhs: right-hand side and initial guess of one implicit step
 *   (step_implicit, timestep.py:155-164): first != 0: rhs = w - q0*f, guess = w;
 *   else rhs = ((2w - wp) + qh*lap) - qd*(f*fs), guess = 2w - wp, lap = c^2 L_h wp.
 * whb_vec_xpay: y = x + a*y  (p = z + beta*p, linalg.py:97).
 * whb_mg_setup / whb_mg_vcycle: 2D all-Dirichlet geometric multigrid for
 *   I - (dt^2/2) c^2 L_h (MultigridHierarchy, linalg.py:189-346): nlev levels,
 *   cells[2*l + a] cells of level l on axis a (level 0 = the context grid, each
 *   level halves both), gamma[2*l + a] = coef/dx_a^2, diag[l] = 1 + 2*sum(gamma),
 *   coarse_inv = inverse of the coarsest interior matrix (row-major, interior
 *   points row-major), nu1/nu2 pre/post red-black sweeps; whb_mg_vcycle:
 *   u = one V-cycle applied to b from u = 0 (the CG preconditioner).
 * whb_tri_setup / whb_tri_solve: 1D Dirichlet tridiagonal elimination
 *   (TridiagFactorization, linalg.py:380-421): n = points - 2 interior unknowns,
 *   sub[n-1], dp[n], cp[n-1] the host factorisation; x = scatter(solve(b interior)). */
int whb_imp_apply(whb_ctx *ctx, int x, int y, double s, int tmp);
int whb_imp_rhs(whb_ctx *ctx, int w, int wp, int lap, int f, int rhs, int guess, int first, double q0,
                double qh, double qd, double fs);
int whb_vec_xpay(whb_ctx *ctx, int x, double a, int y);
int whb_mg_setup(whb_ctx *ctx, int nlev, const int64_t *cells, const double *gamma, const double *diag,
                 const double *coarse_inv, int nu1, int nu2);
int whb_mg_vcycle(whb_ctx *ctx, int b, int u);
int whb_tri_setup(whb_ctx *ctx, int n, const double *sub, const double *dp, const double *cp);
int whb_tri_solve(whb_ctx *ctx, int b, int x);
/* Device-resident CG (cg_solve, linalg.py:62-99) with scalars kept on the device.
 * precond: 0 none (z must be r), 1 multigrid V-cycle, 2 tridiagonal.
 * whb_cg_begin: z = M r, p = z, rz = r.z (device); *rr = r.r.
 * whb_cg_iterate: one iteration — Ap = A p (A = I - s c^2 L_h, tmp as in
 *   whb_imp_apply), alpha = rz/pAp, x += alpha p, r -= alpha Ap, z = M r,
 *   beta = r.z/rz, p = z + beta p — as one CUDA graph; returns *pap = p.Ap and
 *   *rr = r.r.  When pap <= 0 or is not finite nothing is updated (the
 *   reference's breakdown exit). */
int whb_cg_begin(whb_ctx *ctx, int r, int z, int p, int precond, double *rr);
int whb_cg_iterate(whb_ctx *ctx, int x, int r, int z, int p, int ap, int tmp, double s, int precond, double *pap,
                   double *rr);

/* ---- introspection -------------------------------------------------------- */
/* Number of kernel launches issued by this context since creation. */
int whb_launch_count(whb_ctx *ctx, int64_t *count);
/* Per-launch average device time (ms) of the fused step kernel over the last
 * whb_fpi/whb_filtered_solve call when timing is enabled (events on the
 * context stream). */
int whb_set_timing(whb_ctx *ctx, int enable);
int whb_last_timing(whb_ctx *ctx, double *step_kernel_ms_total, int64_t *step_kernel_launches,
                    double *solve_ms_total);
/* Benchmark hygiene: when bytes > 0, whb_fpi writes a scratch buffer of that
 * size (larger than the 126 MB L2) before every pass, outside the timed span. */
int whb_set_l2_flush(whb_ctx *ctx, int64_t bytes);
/* Pinned host buffers for H2D/D2H at full PCIe rate. */
int whb_host_alloc(void **ptr, int64_t bytes);
int whb_host_free(void *ptr);
/* Peer-memory halo exchange between slab ranks (slab.PeerHalo; SURVEY §8(e) "P2P over
 * NVLink" alternative to NCCL send/recv; no reference counterpart — the reference is
 * single-process).  whb_ipc_handle: CUDA IPC handle (64 bytes) of the allocation holding
 * dev_ptr and dev_ptr's byte offset in it; whb_ipc_open / whb_ipc_close map / unmap a peer's
 * allocation in this process.  whb_flags_alloc: `count` zeroed uint32 flags in device memory.
 * whb_copy_async: stream-ordered copy on the context stream, or on the exchange stream inside
 * whb_comm_begin / whb_comm_end (any two device addresses, e.g.
 * local boundary planes -> a neighbour's ghost planes over NVLink).  whb_stream_write_u32 /
 * whb_stream_wait_u32: stream memory operations (write after the stream's earlier work, with
 * a fence; wait until (int32)(*flag - value) >= 0) — the ranks' flags order the exchange
 * without host round trips and without any kernel spinning on the device. */
int whb_ipc_handle(whb_ctx *ctx, uint64_t dev_ptr, void *handle_out, int64_t *offset_out);
int whb_ipc_open(whb_ctx *ctx, const void *handle, uint64_t *base_out);
int whb_ipc_close(whb_ctx *ctx, uint64_t base);
int whb_flags_alloc(whb_ctx *ctx, int count, uint64_t *dev_ptr);
int whb_flags_free(whb_ctx *ctx, uint64_t dev_ptr);
int whb_copy_async(whb_ctx *ctx, uint64_t src_ptr, uint64_t dst_ptr, int64_t bytes);
int whb_stream_write_u32(whb_ctx *ctx, uint64_t dev_ptr, uint32_t value);
int whb_stream_wait_u32(whb_ctx *ctx, uint64_t dev_ptr, uint32_t value);

/* Halo exchange stream (slab.py start/finish).  whb_comm_begin: the context's exchange stream
 * waits for everything enqueued so far (the boundary planes), and whb_copy_async /
 * whb_stream_write_u32 / whb_nccl_exchange go on it until whb_comm_end; whb_comm_join: the
 * context stream waits for that exchange.  Kernels enqueued between end and join (the interior
 * planes) run while the exchange is in flight.  Graph capture follows the fork and join. */
int whb_comm_begin(whb_ctx *ctx);
int whb_comm_end(whb_ctx *ctx);
int whb_comm_join(whb_ctx *ctx);

/* NCCL halo path inside the C ABI (replaces torch.distributed P2P on the data path; libnccl is
 * dlopen'ed, reusing the copy the process already loaded).  whb_nccl_unique_id writes the
 * 128-byte ncclUniqueId (rank 0; the caller broadcasts it), whb_nccl_init creates the context's
 * communicator, whb_nccl_exchange posts n (send, recv) pairs of `counts[i]` doubles with
 * peers[i] as one NCCL group on the exchange stream (inside whb_comm_begin/end; capturable),
 * whb_nccl_allreduce_sum sums one double across the ranks (synchronous). */
int whb_nccl_unique_id(void *id_out);
int whb_nccl_init(whb_ctx *ctx, int nranks, int rank, const void *id);
int whb_nccl_exchange(whb_ctx *ctx, int n, const uint64_t *send_ptrs, const uint64_t *recv_ptrs,
                      const int64_t *counts, const int *peers);
int whb_nccl_allreduce_sum(whb_ctx *ctx, double *value);

/* Caller-captured graphs: whb_capture_begin starts stream capture on the context stream
 * (relaxed mode, so several contexts can capture at once), every later call enqueues into the
 * capture (whb_solve_end then leaves the residual on the device), whb_capture_end instantiates
 * it; whb_graph_launch replays it; whb_resid_read copies the last residual sum to the host.
 * Used for one slab iteration with its peer-memory exchange (slab.PeerSlabGraphs). */
int whb_capture_begin(whb_ctx *ctx);
int whb_capture_end(whb_ctx *ctx, int *graph_id);
int whb_graph_launch(whb_ctx *ctx, int graph_id);
int whb_resid_read(whb_ctx *ctx, double *resid_sq);

/* Launch plan: kernel 0 = simple LDG, 1 = bulk-copy rows (2D/batched), 2 = TMA tensor
 * boxes (3D), 3 = general operator, 4 = cluster-resident small 2D grid (the whole solve,
 * and a whole fixed-point loop, in one launch from shared memory); steps_per_pass = leapfrog
 * steps per HBM pass of the whole-solve kernels (2 two-step, 3/4 wavefront; 0 for kernel 4,
 * which makes no per-step HBM pass).  Step-level (slab) control always uses the multi-pass
 * kernels. */
int whb_plan(whb_ctx *ctx, int *kernel, int *steps_per_pass);
/* Global and local geometry: shape3[3], pitch, nloc (owned planes). */
int whb_geometry(whb_ctx *ctx, int64_t *shape3, int64_t *pitch, int64_t *nloc);

#ifdef __cplusplus
}
#endif
#endif /* WHB200_H */
