/*
 * aderdg_b200.h -- C-ABI of libaderdg_b200.so, the B200 (sm_100a) ADER-DG
 * time step for the compressible Euler equations.
 *
 * The reference (/root/reference/pkg/src/aderdg, arXiv:1808.03788 desk
 * implementation) is pure Python/numpy and has no FFI of its own; its
 * boundary for this path is the Python solver API.  Each entry point below
 * replaces one reference function (file:line cited) and is bound by the
 * drop-in host layer `paper_1808_03788_b200/_lib.py` through ctypes.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers to caller-owned fp64 buffers in
 *    the reference layout: u[cells_0..cells_{d-1}, P (x) .. P (last), m],
 *    quantity fastest (driver.py:131-133, mesh.py:48-63).
 *  - All calls are stream ordered on `stream` (a cudaStream_t) and never
 *    synchronise the host; scalars that change per step (dt, t) live in
 *    device memory so a step sequence is CUDA-graph capturable.
 *  - Return value: ADG_OK or an error code; adg_last_error() describes it.
 *    The host layer maps ADG_ERR_INVALID -> ValueError, ADG_ERR_RUNTIME ->
 *    RuntimeError, ADG_ERR_UNSUPPORTED -> NotImplementedError.
 *  - A handle is bound to one device and is not thread safe.
 */
#ifndef ADERDG_B200_H
#define ADERDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADG_OK 0
#define ADG_ERR_INVALID 1
#define ADG_ERR_RUNTIME 2
#define ADG_ERR_CUDA 3
#define ADG_ERR_UNSUPPORTED 4

/* face kinds, driver.py:23 BOUNDARY_KINDS; ADG_BC_GHOST = exterior trace
 * supplied by the caller (reference "exact" faces, or a neighbour rank's
 * halo under slab decomposition) */
#define ADG_BC_PERIODIC 0
#define ADG_BC_OUTFLOW 1
#define ADG_BC_WALL 2
#define ADG_BC_GHOST 3

/* status word bits written by adg_timestep / adg_update (device int32) */
#define ADG_STATUS_NO_ADMISSIBLE 1   /* corrector.py:44-45 RuntimeError */
#define ADG_STATUS_NONFINITE 2       /* driver.py:197-199 RuntimeError  */

typedef struct adg_handle adg_handle;

/* Grid descriptor (POD).  cells are the LOCAL element counts of this rank;
 * dx are the element widths (mesh.py:32).  dim in 1..3, degree in 0..9,
 * nvars = dim + 2 (Euler) or 1 (advection).  mode = predictor_mode (driver.py:45-48):
 * ADG_MODE_CONSERVATIVE evolves the predictor and the MUSCL-Hancock half
 * step in conservative variables, ADG_MODE_PRIMITIVE in primitive ones
 * (predictor.py:94-96, :165-189; limiter.py:127-177). */
#define ADG_MODE_CONSERVATIVE 0
#define ADG_MODE_PRIMITIVE 1

/* PDE plugin (reference systems.py:355-361 make_system): ADG_SYS_EULER
 * (CompressibleEuler, nvars = dim + 2, gamma) or ADG_SYS_ADVECTION
 * (LinearAdvection, systems.py:77-109: nvars = 1, constant velocity) */
#define ADG_SYS_EULER 0
#define ADG_SYS_ADVECTION 1
/* DiffuseInterfaceElasticity (systems.py:237-345): dim = 2, nvars = 9, a pure
 * nonconservative product with path-conservative faces (corrector.py:65-129) */
#define ADG_SYS_ELASTICITY 2

/* adg_grid.flags.  ADG_GRID_FOLD_STATE: the predictor's volume output is
 * w = u^n + vol / mass (mass = |cell| w_node) instead of the volume integral
 * itself, and adg_update forms u^(n+1) = w - (sum of face terms) / mass from
 * it without reading u^n again (one array less through HBM; the reference's
 * u + (vol - faces) / mass, corrector.py:199-205, re-associated: differences
 * at the 1e-16 level).  Only where adg_fold_supported(g): Euler, conservative
 * predictor, shared-tile kernel (not 3-D N >= 7). */
#define ADG_GRID_FOLD_STATE 1

typedef struct adg_grid {
  int32_t dim;
  int32_t degree;
  int32_t nvars;
  int32_t mode;
  int64_t cells[3];
  double dx[3];
  double gamma;
  int32_t bc[3][2];
  int32_t system;       /* ADG_SYS_* */
  int32_t flags;        /* ADG_GRID_* (0: none) */
  double velocity[3];   /* ADG_SYS_ADVECTION: a_j (unused entries 0) */
} adg_grid;

/* Reduction record filled on device by adg_wavespeed / adg_update and read
 * by adg_timestep: per-axis max |lambda| over admissible nodes as uint64
 * bit patterns of non-negative doubles (max is order independent, so the
 * result is bitwise deterministic), admissible and non-finite counts. */
typedef struct adg_reduce {
  uint64_t lam_bits[3];
  uint64_t n_admissible;
  uint64_t n_nonfinite;
  uint64_t reserved[3];
} adg_reduce;

/* -- lifetime ------------------------------------------------------------ */
int adg_create(int device, adg_handle** out);
int adg_destroy(adg_handle* h);
const char* adg_last_error(const adg_handle* h);
int adg_version(void);

/* Upload the per-degree constants (replaces basis.py:166-202 BasisTables and
 * predictor.py:21-47 TimeOperators).  blob layout (P = degree + 1, S = 2N+1):
 * nodes[P] weights[P] diff[P*P] left[P] right[P] gw[P*P] g0[P] k1_opnorm[1]
 * sub_project[S*P] sub_recover[P*S]; n = total doubles.  Process-wide. */
int adg_set_tables(adg_handle* h, int degree, const double* host_blob, int64_t n);

/* -- corrector.compute_timestep (corrector.py:30-55) --------------------- */
/* zero *red, then fold max |lambda_j| / admissible / non-finite counts of
 * the nodal states u into it */
int adg_wavespeed(adg_handle* h, const adg_grid* g, const double* u, adg_reduce* red,
                  void* stream);
/* dt = min(cfl / sum_j lam_j/dx_j, t_end - t) written to *dt_dev (inf when
 * every speed is zero); sets ADG_STATUS_* bits in *status_dev.  t_dev may be
 * NULL (t = 0). */
int adg_timestep(adg_handle* h, const adg_grid* g, const adg_reduce* red, double cfl,
                 const double* t_dev, double t_end, double* dt_dev, int32_t* status_dev,
                 void* stream);

/* t += dt on device; t_out (may be NULL) receives the new time (the
 * `self.t += trial` of driver.py:175) */
int adg_advance_time(adg_handle* h, double* t_dev, const double* dt_dev, double* t_out,
                     void* stream);

/* History bookkeeping of a device-resident batch (driver.py:344-350 rows):
 * rows[*cnt] = row[0:ncols], status[*cnt] = *status_in, sweeps[*cnt] =
 * max(elem_sweeps[0:n_elem]), then *cnt += 1.  One launch instead of a
 * reduction and three indexed copies per step in the replayed CUDA graph. */
int adg_log_step(adg_handle* h, const double* row, int64_t ncols, const int32_t* status_in,
                 const int32_t* elem_sweeps, int64_t n_elem, double* rows, int32_t* status,
                 int32_t* sweeps, int64_t* cnt, void* stream);

/* -- predictor: startup_guess + picard_solve + extract_traces + the
 *    corrector's volume_integral, fused per element
 *    (predictor.py:99-191, :218-230; corrector.py:141-177) -------------- */
/* u       : nodal states at t_n
 * dt_dev  : device scalar time step
 * tol, max_iter (<=0 -> 2N+2), min_iter: Picard control; an element stops
 *           at its first converged sweep >= min_iter
 * q_out   : optional [E, P^d, P_t, m] space-time predictor (NULL to skip)
 * vol_out : [E, P^d, m] volume accumulator (true integral)
 * traces  : [d][2][E][adg_trace_block(g)] face traces (side 0 = low
 *           face); the block holds P^(d-1) x P_t x m values ordered per
 *           axis x: [j][k][t][v], y: [k][t][i][v], z: [t][i][j][v]
 * pred_bad: [E] uint8, ADG_PRED_* bits; 0 = converged && admissible
 *           (driver.py:212)
 * sweeps  : [E] int32 Picard sweeps taken
 * 3-D N >= 8 grids keep the space-time iterate and its rates in a
 * library-owned HBM workspace of the handle (element batches of at most
 * 28 GiB; grown on the first call, never freed under a captured graph).  */
int adg_predict(adg_handle* h, const adg_grid* g, const double* u, const double* dt_dev,
                double tol, int max_iter, int min_iter, double* q_out, double* vol_out,
                double* traces, uint8_t* pred_bad, int32_t* sweeps, void* stream);

/* pred_bad bits (predictor.py:57-62 PredictorResult flags; any bit set means
 * the element goes to the limiter, driver.py:212) */
#define ADG_PRED_NOT_CONVERGED 1   /* residual above tol at the last sweep */
#define ADG_PRED_INADMISSIBLE 2    /* a converged space-time node is inadmissible */

/* -- picard_solve with the reference's optional arguments
 *    (predictor.py:135-191, :99-126; Euler and advection):
 * q_init  : optional starting iterate [E, P^d, P_t, m] in the iterate
 *           variables (conservative, or primitive in ADG_MODE_PRIMITIVE),
 *           replacing the startup guess (picard_solve initial=); NULL = the
 *           startup guess
 * flags   : ADG_PRED_STARTUP_ONLY -> no sweeps; q_out receives the startup
 *           guess itself in the iterate variables (predictor.startup_guess)
 * other arguments as adg_predict.  Euler runs the shared-tile kernel (its
 * large-tile variant for 3-D N >= 7). */
#define ADG_PRED_STARTUP_ONLY 1
int adg_predict_ex(adg_handle* h, const adg_grid* g, const double* u, const double* q_init,
                   const double* dt_dev, double tol, int max_iter, int min_iter, int flags,
                   double* q_out, double* vol_out, double* traces, uint8_t* pred_bad,
                   int32_t* sweeps, void* stream);

/* -- predictor.extract_traces (predictor.py:218-230) of a given space-time
 *    q [E, P^d, P_t, m]: out [d][2 sides][E][P^(d-1) tangential][P_t][m]
 *    (tangential axes ascending, side 0 = phi(0)); any system (linear) */
int adg_extract_traces(adg_handle* h, const adg_grid* g, const double* q, double* out,
                       void* stream);

/* -- the space-time rate L(q) at every node of q [E, P^d, P_t, m] (Euler,
 *    advection): conservative -sum_j (D/dx_j) F_j(q) in _rhs_conservative's order
 *    (predictor.py:74-91), or primitive_rhs(v, grad v) for
 *    ADG_MODE_PRIMITIVE (q holds primitive states, predictor.py:94-96).
 *    The building block of weak_form_defect (predictor.py:194-215). */
int adg_spacetime_rate(adg_handle* h, const adg_grid* g, const double* q, double* rate,
                       void* stream);

/* -- the same predictor on the element range [e_begin, e_begin + e_count)
 *    of the grid (element order = the reference's C order of `u`).  u,
 *    vol_out, traces, pred_bad, sweeps (and q_out) are the WHOLE grid's
 *    arrays; only the range's entries are written.  Results are bitwise
 *    those of adg_predict (per-element arithmetic).  Used by the slab
 *    decomposition to predict the two boundary layers first and overlap
 *    their halo exchange with the interior (no reference counterpart: the
 *    reference is single-process).  ADG_ERR_UNSUPPORTED unless
 *    adg_predict_range_supported(g) (3-D N >= 7 conservative grids run the
 *    whole-grid phased / slice-streaming predictors). */
int adg_predict_range(adg_handle* h, const adg_grid* g, int64_t e_begin, int64_t e_count,
                      const double* u, const double* dt_dev, double tol, int max_iter,
                      int min_iter, double* q_out, double* vol_out, double* traces,
                      uint8_t* pred_bad, int32_t* sweeps, void* stream);
int adg_predict_range_supported(const adg_grid* g);
/* 1 if this grid's predictor / update pair implements ADG_GRID_FOLD_STATE */
int adg_fold_supported(const adg_grid* g);

/* -- face coupling along one axis: driver._face_states (driver.py:234-261)
 *    + corrector.face_fluxes (corrector.py:100-129) + the time weighting of
 *    face_integral (corrector.py:186) ------------------------------------ */
/* fd: element-major face terms [E][d axes][2 sides][P^(d-1)][m] shared by
 * all axes; this call fills the entries of `axis` with the time-integrated
 * low-side Rusanov term sum_t w_t d_low of each face (for the element's
 * high face, and for the low face of the element above it, where the
 * high-side term is its exact negation).  Traces are the predictor's blocks;
 * ghost_lo / ghost_hi: exterior trace blocks for ADG_BC_GHOST faces,
 * [cells with 1 along axis][trace block], else NULL. */
int adg_face_flux(adg_handle* h, const adg_grid* g, int axis, const double* traces,
                  const double* ghost_lo, const double* ghost_hi, double* fd,
                  void* stream);

/* -- corrector.face_integral + element_update (corrector.py:180-205) with a
 *    fused epilogue: wave speeds of u_out folded into red_next (the next
 *    step's compute_timestep) and per-block conserved-total partials
 *    (driver.py:344-350).  fd filled by adg_face_flux for every axis.
 *    u, vol, fd stream through TMA bulk copies (16-byte aligned buffers).
 *    totals_partial: [adg_update_blocks(g), m] (may be NULL).            */
int adg_update(adg_handle* h, const adg_grid* g, const double* u, const double* vol,
               const double* fd, const double* dt_dev, double* u_out, adg_reduce* red_next,
               double* totals_partial, void* stream);
int64_t adg_update_blocks(const adg_grid* g);
/* doubles per element trace block: P^d m rounded up to even (16-byte
 * multiple, so the face kernel moves each block with one TMA bulk copy);
 * traces are [d][2][E][adg_trace_block(g)], ghost planes likewise */
int64_t adg_trace_block(const adg_grid* g);
/* totals[m] = cell_volume * fixed-order sum of the partials */
int adg_totals_finalize(adg_handle* h, const adg_grid* g, const double* totals_partial,
                        int64_t nblocks, double* totals_out, void* stream);

/* conserved totals of u directly (driver.py:344-350); partial has
 * adg_update_blocks(g) * m doubles */
int adg_totals(adg_handle* h, const adg_grid* g, const double* u, double* partial,
               double* totals_out, void* stream);

/* adg_wavespeed and adg_totals of the same state in ONE pass over u (the
 * limited step re-records a state the rescue changed: corrector.py:30-55 and
 * driver.py:344-350 together); results bitwise those of the two calls */
int adg_state_record(adg_handle* h, const adg_grid* g, const double* u, adg_reduce* red,
                     double* partial, double* totals_out, void* stream);

/* -- a posteriori subcell limiter (limiter.py; driver.py:265-299) ------- */
/* Exterior subcell averages for ADG_BC_GHOST ("exact") faces, the
 * reference's _boundary_slab (driver.py:317-340) evaluated by the caller at
 * t_n: slab[j][s] (device, NULL for other faces) holds `layers` subcell layers
 * beyond face (j, s) as [len_0]..[len_{d-1}][m], len_i = n_i S + 2 layers
 * for i < j (the axes padded before j, corners included), layers for i = j
 * (outward order: index 0 is the farthest layer on side 0, the nearest on
 * side 1), n_i S for i > j; layers >= max(S, 2). */
typedef struct adg_subcell_ghosts {
  const double* slab[3][2];
  int32_t layers;
  int32_t reserved;
} adg_subcell_ghosts;

/* Subcell averages of u^n (limiter.project_to_subcells, limiter.py:27-33)
 * sub_out [E, S^d, m] (S = 2N+1) and their per-cell extrema cmin/cmax
 * [E, m] (the per-cell part of limiter.relaxed_bounds, limiter.py:62-63).
 * Device limiter: every dimension and degree (3-D windows beyond shared
 * memory run on L2-resident global scratch). */
int adg_project_subcells(adg_handle* h, const adg_grid* g, const double* u, double* sub_out,
                         double* cmin_out, double* cmax_out, void* stream);
/* Troubled-cell detection (limiter.py:51-86 + driver.py:272-285): DMP
 * bounds from the own and 2d face-neighbour cells of prev_sub (ghost cells
 * through the face kinds, driver.py:301-340), relaxed by
 * max(delta0, eps (hi - lo)); a cell is troubled if a candidate subcell
 * average leaves them, a candidate nodal or subcell state is inadmissible,
 * pred_bad is set, or force_all != 0.  Writes troubled[E] (uint8), the
 * compacted list idx[*count] (int32, unordered) and *count (int32).
 * ghosts: exterior slabs of ADG_BC_GHOST faces (NULL if there are none).
 * cand_sub_out / cand_cmin_out / cand_cmax_out (may be NULL): the
 * candidate's subcell averages and extrema; for every cell the rescue
 * leaves alone they are the next step's prev_sub / cmin / cmax. */
int adg_detect(adg_handle* h, const adg_grid* g, const double* prev_sub, const double* cmin,
               const double* cmax, const double* cand, const uint8_t* pred_bad, double delta0,
               double eps, int force_all, const adg_subcell_ghosts* ghosts, uint8_t* troubled,
               int32_t* idx, int32_t* count, double* cand_sub_out, double* cand_cmin_out,
               double* cand_cmax_out, void* stream);
/* MUSCL-Hancock rescue of the listed cells from t^n subcell averages
 * (limiter.py:89-223 + driver.py:286-298), writing recovered nodal states
 * into u_out for listed cells (other cells untouched) and setting
 * *failed_dev != 0 if any cell failed after the first-order retry
 * (driver.py:292-293 restart).  sub_next / cmin_next / cmax_next (may be
 * NULL) receive the rescued cells' subcell averages and extrema, completing
 * adg_detect's candidate outputs into the next step's prev_sub. */
int adg_rescue(adg_handle* h, const adg_grid* g, const double* prev_sub, const int32_t* idx,
               const int32_t* count_dev, int32_t count_host_max, const double* dt_dev,
               const adg_subcell_ghosts* ghosts, double* u_out, int32_t* failed_dev,
               double* sub_next, double* cmin_next, double* cmax_next, void* stream);
/* IC flattening (driver.py:137-152): cells whose nodal or subcell states are
 * inadmissible are replaced by their weighted mean; *nflat = count */
int adg_flatten_ic(adg_handle* h, const adg_grid* g, double* u, int32_t* nflat,
                   void* stream);

/* -- limiter module helpers with the reference's array interfaces
 *    (limiter.py:45-101); Simulation uses the fused adg_detect / adg_rescue */
/* minmod (limiter.py:45-48), elementwise over n doubles */
int adg_minmod(adg_handle* h, int64_t n, const double* a, const double* b, double* out,
               void* stream);
/* relaxed_bounds (limiter.py:51-73): padded_sub [(cells_j + 2)..][nsub][m]
 * (nsub = S^d subcells per cell) -> lo, hi [cells..][m]; cmin_pad / cmax_pad
 * are scratch of (prod (cells_j + 2)) m doubles; cells is a host int64[dim] */
int adg_relaxed_bounds(adg_handle* h, int dim, int nvars, const int64_t* cells, int nsub,
                       const double* padded_sub, double delta0, double eps, double* cmin_pad,
                       double* cmax_pad, double* lo_out, double* hi_out, void* stream);
/* detect_troubled (limiter.py:76-86): cand [E][P^d][m], cand_sub [E][S^d][m],
 * lo / hi [E][m] -> troubled [E] uint8 (E, dim, degree, system from g) */
int adg_detect_cells(adg_handle* h, const adg_grid* g, const double* cand,
                     const double* cand_sub, const double* lo, const double* hi,
                     uint8_t* troubled, void* stream);
/* gather_windows (limiter.py:89-101): padded [padded_dims..][m] (host
 * int64[dim]), starts [nwin][dim] (device int64) -> out [nwin][size^dim][m] */
int adg_gather_windows(adg_handle* h, int dim, int nvars, const int64_t* padded_dims,
                       const double* padded, const int64_t* starts, int64_t nwin, int size,
                       double* out, void* stream);

/* -- module-level pieces: the reference's corrector / limiter functions on
 *    arrays in the reference layouts (element grid flattened: E = product
 *    of g->cells), for callers of the module API rather than Simulation.
 *    dt_dev is a device scalar.  -------------------------------------------- */
/* corrector.face_fluxes (corrector.py:100-129): n point pairs [n][m] ->
 * d_low, d_high [n][m] across a face with normal +e_axis */
int adg_face_fluxes(adg_handle* h, const adg_grid* g, int axis, int64_t n, const double* q_minus,
                    const double* q_plus, double* d_low, double* d_high, void* stream);
/* Pointwise face terms for n state pairs [n][m] and a general unit normal
 * (host double[3]) -- corrector.riemann_dminus (corrector.py:81-97, mode 0:
 * out_a = D(q-, q+).n for the element with outward normal n), face_fluxes
 * (mode 1: out_a = d_low, out_b = d_high for n = e_axis, corrector.py:100-129)
 * -- and, for the nonconservative system, path_integral_B (corrector.py:65-78):
 * bpath [n][m][m] (may be NULL; mode -1 computes only it).  Euler, advection
 * and elasticity-di. */
/* mode 2 (Euler, advection): out_a [n] = rusanov_theta (corrector.py:58-62),
 * the larger |eigenvalue . n| of the two states (NaN propagates) */
int adg_riemann_points(adg_handle* h, const adg_grid* g, int64_t n, const double* normal,
                       int mode, const double* q_minus, const double* q_plus, double* out_a,
                       double* out_b, double* bpath, void* stream);
/* corrector.volume_integral (corrector.py:141-177): q [E][P^d][P_t][m] ->
 * vol [E][P^d][m] */
int adg_volume_integral(adg_handle* h, const adg_grid* g, const double* q, const double* dt_dev,
                        double* vol_out, void* stream);
/* corrector.face_integral (corrector.py:180-196): d_values
 * [E][P^(d-1) tangential][P_t][m] of face (axis, side) -> [E][P^d][m] */
int adg_face_integral(adg_handle* h, const adg_grid* g, int axis, int side,
                      const double* d_values, const double* dt_dev, double* out, void* stream);
/* corrector.element_update (corrector.py:199-205): u + (vol - acc_0 - ..)
 * / mass; accs is a host array of n_acc (<= 6) device pointers */
int adg_element_update(adg_handle* h, const adg_grid* g, const double* u, const double* vol,
                       const double* const* accs, int n_acc, double* u_out, void* stream);
/* limiter.muscl_subcell_step (limiter.py:104-121) on caller windows
 * [T][(S+4)^d][m] (count_dev: device int32 holding T): new averages
 * [T][S^d][m], failed[T] (uint8).  Here g->dx are the SUBCELL widths and
 * g->mode selects the conservative / primitive half step. */
int adg_muscl_windows(adg_handle* h, const adg_grid* g, const double* windows, int64_t n_windows,
                      const int32_t* count_dev, const double* dt_dev, double* avg_out,
                      uint8_t* failed, void* stream);
/* limiter.recover_from_subcells (limiter.py:36-42): [E][S^d][m] -> [E][P^d][m] */
int adg_recover_subcells(adg_handle* h, const adg_grid* g, const double* ubar, double* u_out,
                         void* stream);
/* limiter.flatten_inadmissible (limiter.py:205-223), in place on nodal
 * [E][P^d][m] with the cells' averages [E][S^d][m]; *nflat = cells flattened */
int adg_flatten_cells(adg_handle* h, const adg_grid* g, double* nodal, const double* averages,
                      int32_t* nflat, void* stream);

/* -- multi-GPU exchange of the x-slab decomposition (
 *    the reference is single-process, driver.py:186-248): an NCCL
 *    communicator bound to a handle's device, one rank per GPU.  All calls
 *    are stream ordered on `stream` and CUDA-graph capturable. ------------ */
typedef struct adg_comm adg_comm;
#define ADG_COMM_ID_BYTES 128
/* rank 0 creates the id (ncclGetUniqueId) and shares the bytes with the other
 * ranks out of band (the host layer uses torch.distributed.broadcast) */
int adg_comm_unique_id(void* id_out);
int adg_comm_init(adg_handle* h, const void* id, int nranks, int rank, adg_comm** out);
int adg_comm_destroy(adg_comm* c);
/* Face-trace halo swap along x on the periodic ring of ranks (the
 * reference's periodic face states across the slab cut, driver.py:234-248):
 * sends the low-x trace plane of the first element layer to rank-1 and the
 * high-x plane of the last layer to rank+1 (grouped ncclSend / ncclRecv);
 * ghost_lo / ghost_hi receive the neighbours' planes ([cells_y cells_z]
 * trace blocks, the ADG_BC_GHOST data of adg_face_flux).  traces as
 * adg_predict writes them. */
int adg_halo_exchange(adg_handle* h, adg_comm* c, const adg_grid* g, const double* traces,
                      double* ghost_lo, double* ghost_hi, void* stream);
/* The global CFL record (corrector.py:47-55 over all ranks): MAX of the
 * per-axis wave-speed bit patterns, SUM of the admissible / non-finite
 * counts, in place. */
int adg_allreduce_reduce(adg_handle* h, adg_comm* c, adg_reduce* red, void* stream);
/* SUM of n doubles in place (conserved totals rows, driver.py:344-350). */
int adg_allreduce_sum(adg_handle* h, adg_comm* c, double* buf, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ADERDG_B200_H */
