// adg_api.cu -- extern "C" entry points of libaderdg_b200.so.
// Each maps onto one reference function; see include/aderdg_b200.h.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {
__constant__ DegreeTables c_tab[kMaxP];
DegreeTables h_tab[kMaxP];

void upload_tables(int degree, const double* blob, int64_t n, std::string* err, int* rc) {
  const int P = degree + 1, S = 2 * degree + 1;
  const int64_t need = 5 * P + 2 * P * P + 1 + 2 * S * P;
  if (degree < 0 || degree > 9 || n != need) {
    *err = "bad table blob (degree " + std::to_string(degree) + ", n=" + std::to_string(n) +
           ", need " + std::to_string(need) + ")";
    *rc = ADG_ERR_INVALID;
    return;
  }
  DegreeTables t;
  std::memset(&t, 0, sizeof(t));
  const double* p = blob;
  std::memcpy(t.nodes, p, P * 8); p += P;
  std::memcpy(t.weights, p, P * 8); p += P;
  std::memcpy(t.diff, p, P * P * 8); p += P * P;
  std::memcpy(t.left, p, P * 8); p += P;
  std::memcpy(t.right, p, P * 8); p += P;
  std::memcpy(t.gw, p, P * P * 8); p += P * P;
  std::memcpy(t.g0, p, P * 8); p += P;
  t.k1_opnorm = *p; p += 1;
  std::memcpy(t.sub_project, p, S * P * 8); p += S * P;
  std::memcpy(t.sub_recover, p, P * S * 8); p += P * S;
  // stiff[k, l] = diff[l, k] * w[l]  ((diff * w[:, None]).T, corrector.py:168)
  for (int k = 0; k < P; ++k)
    for (int l = 0; l < P; ++l) t.stiff[k * P + l] = t.diff[l * P + k] * t.weights[l];
  t.loaded = 1;
  h_tab[degree] = t;
  cudaError_t ce = cudaMemcpyToSymbol(c_tab, &t, sizeof(t), sizeof(t) * degree);
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    *rc = ADG_ERR_CUDA;
    return;
  }
  *rc = ADG_OK;
}
}  // namespace adg

struct adg_handle {
  int device = 0;
  int num_sms = 148;
  std::string err;
  bool tables_loaded[10] = {false};
  // predictor global-tile workspace (large 3-D tiles).  It only grows, and a
  // buffer it outgrows is retired (freed at adg_destroy), never freed while a
  // captured CUDA graph may still hold its address.
  double* ws = nullptr;
  size_t ws_bytes = 0;
  std::vector<double*> retired;
};

// Every entry point runs on the handle's device and restores the caller's
// current device on return (a handle is bound to one device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const adg_handle* h) {
    if (!h) return;
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != h->device &&
        cudaSetDevice(h->device) == cudaSuccess)
      prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

static int grow_workspace(adg_handle* h, size_t need) {
  if (need <= h->ws_bytes) return ADG_OK;
  double* p = nullptr;
  if (cudaMalloc(&p, need) != cudaSuccess) {
    h->err = "cannot allocate predictor workspace";
    return ADG_ERR_CUDA;
  }
  if (h->ws) h->retired.push_back(h->ws);
  h->ws = p;
  h->ws_bytes = need;
  return ADG_OK;
}

static int fail(adg_handle* h, int rc, const std::string& msg) {
  if (h) h->err = msg;
  return rc;
}

static int check_grid(adg_handle* h, const adg_grid* g) {
  if (!g) return fail(h, ADG_ERR_INVALID, "null grid");
  if (g->dim < 1 || g->dim > 3) return fail(h, ADG_ERR_INVALID, "dim must be 1..3");
  if (g->degree < 0 || g->degree > 9) return fail(h, ADG_ERR_INVALID, "degree must be 0..9");
  if (g->system == ADG_SYS_ADVECTION) {
    if (g->nvars != 1) return fail(h, ADG_ERR_INVALID, "advection has m = 1");
    if (g->mode != ADG_MODE_CONSERVATIVE)
      return fail(h, ADG_ERR_UNSUPPORTED, "advection on the device: conservative predictor only");
  } else if (g->system == ADG_SYS_ELASTICITY) {
    if (g->dim != 2) return fail(h, ADG_ERR_INVALID, "elasticity-di is 2-D");
    if (g->nvars != 9) return fail(h, ADG_ERR_INVALID, "elasticity-di has m = 9");
    if (g->mode != ADG_MODE_CONSERVATIVE)
      return fail(h, ADG_ERR_UNSUPPORTED,
                  "elasticity-di on the device: conservative predictor only");
  } else if (g->system != ADG_SYS_EULER) {
    return fail(h, ADG_ERR_UNSUPPORTED, "unknown system");
  } else if (g->nvars != g->dim + 2) {
    return fail(h, ADG_ERR_INVALID, "Euler has m = d + 2");
  }
  for (int j = 0; j < g->dim; ++j) {
    if (g->cells[j] < 1) return fail(h, ADG_ERR_INVALID, "cell counts must be positive");
    if (!(g->dx[j] > 0.0)) return fail(h, ADG_ERR_INVALID, "spacings must be positive");
    for (int s = 0; s < 2; ++s)
      if (g->bc[j][s] < 0 || g->bc[j][s] > 3) return fail(h, ADG_ERR_INVALID, "bad bc kind");
  }
  if (!h->tables_loaded[g->degree])
    return fail(h, ADG_ERR_INVALID, "tables for this degree not uploaded (adg_set_tables)");
  if (g->flags & ~ADG_GRID_FOLD_STATE) return fail(h, ADG_ERR_INVALID, "unknown grid flags");
  if ((g->flags & ADG_GRID_FOLD_STATE) &&
      (g->system != ADG_SYS_EULER || !adg::predict_fold_supported(g)))
    return fail(h, ADG_ERR_UNSUPPORTED,
                "ADG_GRID_FOLD_STATE: not supported for this grid (adg_fold_supported)");
  return ADG_OK;
}

static bool is_adv(const adg_grid* g) { return g && g->system == ADG_SYS_ADVECTION; }
static bool is_el(const adg_grid* g) { return g && g->system == ADG_SYS_ELASTICITY; }

// entry points with Euler kernels only (limiter, module-level pieces)
static int check_euler(adg_handle* h, const adg_grid* g) {
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (is_adv(g) || is_el(g))
    return fail(h, ADG_ERR_UNSUPPORTED,
                "advection / elasticity-di on the device: the limiter and the module-level "
                "pieces are Euler only");
  return ADG_OK;
}

// limiter entry points: the kernels carry Euler and advection policies
static int check_limiter(adg_handle* h, const adg_grid* g) {
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (is_el(g))
    return fail(h, ADG_ERR_UNSUPPORTED,
                "elasticity-di on the device: no subcell limiter (Euler and advection)");
  return ADG_OK;
}

static int wrap(adg_handle* h, int rc, const std::string& e) {
  if (rc != ADG_OK) h->err = e;
  return rc;
}

extern "C" {

int adg_version(void) { return 1; }

int adg_create(int device, adg_handle** out) {
  if (!out) return ADG_ERR_INVALID;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return ADG_ERR_CUDA;
  adg_handle* h = new adg_handle();
  h->device = device;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  *out = h;
  return ADG_OK;
}

int adg_destroy(adg_handle* h) {
  if (!h) return ADG_OK;
  DeviceGuard dg(h);
  if (h->ws) cudaFree(h->ws);
  for (double* p : h->retired) cudaFree(p);
  delete h;
  return ADG_OK;
}

const char* adg_last_error(const adg_handle* h) { return h ? h->err.c_str() : "null handle"; }

int adg_set_tables(adg_handle* h, int degree, const double* host_blob, int64_t n) {
  DeviceGuard dg(h);
  if (!h || !host_blob) return ADG_ERR_INVALID;
  std::string e;
  int rc = ADG_OK;
  adg::upload_tables(degree, host_blob, n, &e, &rc);
  if (rc == ADG_OK) h->tables_loaded[degree] = true;
  return wrap(h, rc, e);
}

int adg_wavespeed(adg_handle* h, const adg_grid* g, const double* u, adg_reduce* red,
                  void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  std::string e;
  if (is_adv(g))
    return wrap(h, adg::adv_state_reduce(g, u, red, nullptr, (cudaStream_t)stream, &e), e);
  if (is_el(g))
    return wrap(h, adg::el_state_reduce(g, u, red, nullptr, (cudaStream_t)stream, &e), e);
  return wrap(h, adg::state_reduce(g, u, red, nullptr, (cudaStream_t)stream, &e), e);
}

int adg_timestep(adg_handle* h, const adg_grid* g, const adg_reduce* red, double cfl,
                 const double* t_dev, double t_end, double* dt_dev, int32_t* status_dev,
                 void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (!(cfl < 1.0 / (2 * g->degree + 1)))
    return fail(h, ADG_ERR_INVALID, "cfl violates the stability bound 1/(2N+1)");
  std::string e;
  return wrap(h, adg::timestep(g, red, cfl, t_dev, t_end, dt_dev, status_dev,
                               (cudaStream_t)stream, &e), e);
}

int adg_advance_time(adg_handle* h, double* t_dev, const double* dt_dev, double* t_out,
                     void* stream) {
  DeviceGuard dg(h);
  if (!h || !t_dev || !dt_dev) return ADG_ERR_INVALID;
  std::string e;
  return wrap(h, adg::advance_time(t_dev, dt_dev, t_out, (cudaStream_t)stream, &e), e);
}

int adg_log_step(adg_handle* h, const double* row, int64_t ncols, const int32_t* status_in,
                 const int32_t* elem_sweeps, int64_t n_elem, double* rows, int32_t* status,
                 int32_t* sweeps, int64_t* cnt, void* stream) {
  DeviceGuard dg(h);
  if (!h || !row || !status_in || !elem_sweeps || !rows || !status || !sweeps || !cnt ||
      ncols < 0 || n_elem < 1)
    return fail(h, ADG_ERR_INVALID, "adg_log_step: bad arguments");
  std::string e;
  return wrap(h, adg::log_step(row, ncols, status_in, elem_sweeps, n_elem, rows, status, sweeps,
                               cnt, (cudaStream_t)stream, &e), e);
}

int adg_predict(adg_handle* h, const adg_grid* g, const double* u, const double* dt_dev,
                double tol, int max_iter, int min_iter, double* q_out, double* vol_out,
                double* traces, uint8_t* pred_bad, int32_t* sweeps, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  rc = grow_workspace(h, adg::predict_workspace_bytes(g->dim, g->degree + 1, h->num_sms, adg::n_elements(g)));
  if (rc) return rc;
  std::string e;
  if (is_adv(g))
    return wrap(h, adg::adv_predict(g, u, dt_dev, tol, max_iter, min_iter, q_out, vol_out,
                                    traces, pred_bad, sweeps, (cudaStream_t)stream,
                                    h->num_sms, &e), e);
  if (is_el(g))
    return wrap(h, adg::el_predict(g, u, dt_dev, tol, max_iter, min_iter, q_out, vol_out,
                                   traces, pred_bad, sweeps, (cudaStream_t)stream,
                                   h->num_sms, &e), e);
  return wrap(h, adg::predict(g, u, dt_dev, tol, max_iter, min_iter, q_out, vol_out, traces,
                              pred_bad, sweeps, (cudaStream_t)stream, h->num_sms, h->ws,
                              h->ws_bytes, &e), e);
}

int adg_predict_ex(adg_handle* h, const adg_grid* g, const double* u, const double* q_init,
                   const double* dt_dev, double tol, int max_iter, int min_iter, int flags,
                   double* q_out, double* vol_out, double* traces, uint8_t* pred_bad,
                   int32_t* sweeps, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (flags & ~ADG_PRED_STARTUP_ONLY) return fail(h, ADG_ERR_INVALID, "unknown predictor flags");
  std::string e;
  if (is_adv(g))
    return wrap(h, adg::adv_predict(g, u, dt_dev, tol, max_iter, min_iter, q_out, vol_out,
                                    traces, pred_bad, sweeps, (cudaStream_t)stream, h->num_sms,
                                    &e, q_init, (flags & ADG_PRED_STARTUP_ONLY) ? 1 : 0), e);
  if (is_el(g))
    return fail(h, ADG_ERR_UNSUPPORTED,
                "elasticity-di on the device: no starting iterate / startup-only predictor");
  rc = grow_workspace(h, adg::predict_workspace_bytes(g->dim, g->degree + 1, h->num_sms, adg::n_elements(g)));
  if (rc) return rc;
  return wrap(h, adg::predict(g, u, dt_dev, tol, max_iter, min_iter, q_out, vol_out, traces,
                              pred_bad, sweeps, (cudaStream_t)stream, h->num_sms, h->ws,
                              h->ws_bytes, &e, 0, -1, q_init,
                              (flags & ADG_PRED_STARTUP_ONLY) ? 1 : 0), e);
}

int adg_extract_traces(adg_handle* h, const adg_grid* g, const double* q, double* out,
                       void* stream) {
  DeviceGuard dg(h);
  // linear in q: any number of quantities, no plugin
  if (!g || g->dim < 1 || g->dim > 3 || g->degree < 0 || g->degree > 9 || g->nvars < 1 ||
      g->cells[0] < 0)
    return fail(h, ADG_ERR_INVALID, "adg_extract_traces: bad grid");
  if (!h->tables_loaded[g->degree])
    return fail(h, ADG_ERR_INVALID, "tables for this degree not uploaded (adg_set_tables)");
  if (!q || !out) return fail(h, ADG_ERR_INVALID, "adg_extract_traces: null array");
  std::string e;
  return wrap(h, adg::extract_traces(g, q, out, (cudaStream_t)stream, &e), e);
}

int adg_spacetime_rate(adg_handle* h, const adg_grid* g, const double* q, double* rate,
                       void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (!q || !rate) return fail(h, ADG_ERR_INVALID, "adg_spacetime_rate: null array");
  std::string e;
  if (is_adv(g)) return wrap(h, adg::adv_spacetime_rate(g, q, rate, (cudaStream_t)stream, &e), e);
  if (is_el(g)) return fail(h, ADG_ERR_UNSUPPORTED, "adg_spacetime_rate: Euler and advection");
  return wrap(h, adg::spacetime_rate(g, q, rate, (cudaStream_t)stream, &e), e);
}

int adg_fold_supported(const adg_grid* g) {
  return g && !is_adv(g) && !is_el(g) && g->dim >= 1 && g->dim <= 3 &&
                 adg::predict_fold_supported(g)
             ? 1
             : 0;
}

int adg_predict_range_supported(const adg_grid* g) {
  return g && !is_adv(g) && !is_el(g) && adg::predict_range_supported(g) ? 1 : 0;
}

int adg_predict_range(adg_handle* h, const adg_grid* g, int64_t e_begin, int64_t e_count,
                      const double* u, const double* dt_dev, double tol, int max_iter,
                      int min_iter, double* q_out, double* vol_out, double* traces,
                      uint8_t* pred_bad, int32_t* sweeps, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (!adg_predict_range_supported(g))
    return fail(h, ADG_ERR_UNSUPPORTED, "adg_predict_range: grid runs a whole-grid predictor");
  rc = grow_workspace(h, adg::predict_workspace_bytes(g->dim, g->degree + 1, h->num_sms, adg::n_elements(g)));
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::predict(g, u, dt_dev, tol, max_iter, min_iter, q_out, vol_out, traces,
                              pred_bad, sweeps, (cudaStream_t)stream, h->num_sms, h->ws,
                              h->ws_bytes, &e, e_begin, e_count), e);
}

int adg_face_flux(adg_handle* h, const adg_grid* g, int axis, const double* traces,
                  const double* ghost_lo, const double* ghost_hi, double* dbar_out,
                  void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  std::string e;
  if (is_adv(g))
    return wrap(h, adg::adv_face_flux(g, axis, traces, ghost_lo, ghost_hi, dbar_out,
                                      (cudaStream_t)stream, &e), e);
  if (is_el(g))
    return wrap(h, adg::el_face_flux(g, axis, traces, ghost_lo, ghost_hi, dbar_out,
                                     (cudaStream_t)stream, &e), e);
  return wrap(h, adg::face_flux(g, axis, traces, ghost_lo, ghost_hi, dbar_out,
                                (cudaStream_t)stream, &e), e);
}

int64_t adg_update_blocks(const adg_grid* g) { return adg::update_blocks(g); }

int64_t adg_trace_block(const adg_grid* g) {
  int64_t pd = 1;
  for (int j = 0; j < g->dim; ++j) pd *= g->degree + 1;
  const int64_t b = pd * (g->system == ADG_SYS_ADVECTION ? 1
                          : (g->system == ADG_SYS_ELASTICITY ? 9 : g->dim + 2));
  return b + (b & 1);
}

int adg_update(adg_handle* h, const adg_grid* g, const double* u, const double* vol,
               const double* fd, const double* dt_dev, double* u_out, adg_reduce* red_next,
               double* totals_partial, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  std::string e;
  if (is_adv(g))
    return wrap(h, adg::adv_update(g, u, vol, fd, dt_dev, u_out, red_next, totals_partial,
                                   (cudaStream_t)stream, &e), e);
  if (is_el(g))
    return wrap(h, adg::el_update(g, u, vol, fd, dt_dev, u_out, red_next, totals_partial,
                                  (cudaStream_t)stream, &e), e);
  return wrap(h, adg::update(g, u, vol, fd, dt_dev, u_out, red_next, totals_partial,
                             (cudaStream_t)stream, &e), e);
}

int adg_totals_finalize(adg_handle* h, const adg_grid* g, const double* totals_partial,
                        int64_t nblocks, double* totals_out, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::totals_finalize(g, totals_partial, nblocks, totals_out,
                                      (cudaStream_t)stream, &e), e);
}

int adg_totals(adg_handle* h, const adg_grid* g, const double* u, double* partial,
               double* totals_out, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  std::string e;
  rc = is_adv(g)  ? adg::adv_state_reduce(g, u, nullptr, partial, (cudaStream_t)stream, &e)
       : is_el(g) ? adg::el_state_reduce(g, u, nullptr, partial, (cudaStream_t)stream, &e)
                  : adg::state_reduce(g, u, nullptr, partial, (cudaStream_t)stream, &e);
  if (rc) return wrap(h, rc, e);
  return wrap(h, adg::totals_finalize(g, partial, adg::reduce_blocks(g), totals_out,
                                      (cudaStream_t)stream, &e), e);
}

int adg_state_record(adg_handle* h, const adg_grid* g, const double* u, adg_reduce* red,
                     double* partial, double* totals_out, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (!red || !partial || !totals_out)
    return fail(h, ADG_ERR_INVALID, "adg_state_record: null array");
  std::string e;
  rc = is_adv(g)  ? adg::adv_state_reduce(g, u, red, partial, (cudaStream_t)stream, &e)
       : is_el(g) ? adg::el_state_reduce(g, u, red, partial, (cudaStream_t)stream, &e)
                  : adg::state_reduce(g, u, red, partial, (cudaStream_t)stream, &e);
  if (rc) return wrap(h, rc, e);
  return wrap(h, adg::totals_finalize(g, partial, adg::reduce_blocks(g), totals_out,
                                      (cudaStream_t)stream, &e), e);
}

int adg_project_subcells(adg_handle* h, const adg_grid* g, const double* u, double* sub_out,
                         double* cmin_out, double* cmax_out, void* stream) {
  DeviceGuard dg(h);
  int rc = check_limiter(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::project_subcells(g, u, sub_out, cmin_out, cmax_out, (cudaStream_t)stream,
                                       &e), e);
}

int adg_detect(adg_handle* h, const adg_grid* g, const double* prev_sub, const double* cmin,
               const double* cmax, const double* cand, const uint8_t* pred_bad, double delta0,
               double eps, int force_all, const adg_subcell_ghosts* ghosts, uint8_t* troubled,
               int32_t* idx, int32_t* count, double* cand_sub_out, double* cand_cmin_out,
               double* cand_cmax_out, void* stream) {
  DeviceGuard dg(h);
  int rc = check_limiter(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::detect(g, prev_sub, cmin, cmax, cand, pred_bad, delta0, eps, force_all,
                             ghosts, troubled, idx, count, cand_sub_out, cand_cmin_out,
                             cand_cmax_out, (cudaStream_t)stream, &e), e);
}

int adg_rescue(adg_handle* h, const adg_grid* g, const double* prev_sub, const int32_t* idx,
               const int32_t* count_dev, int32_t count_host_max, const double* dt_dev,
               const adg_subcell_ghosts* ghosts, double* u_out, int32_t* failed_dev,
               double* sub_next, double* cmin_next, double* cmax_next, void* stream) {
  DeviceGuard dg(h);
  int rc = check_limiter(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::rescue(g, prev_sub, idx, count_dev, count_host_max, dt_dev, ghosts, u_out,
                             failed_dev, sub_next, cmin_next, cmax_next, (cudaStream_t)stream,
                             &e), e);
}

int adg_face_fluxes(adg_handle* h, const adg_grid* g, int axis, int64_t n, const double* q_minus,
                    const double* q_plus, double* d_low, double* d_high, void* stream) {
  DeviceGuard dg(h);
  int rc = check_euler(h, g);
  if (rc) return rc;
  if (axis < 0 || axis >= g->dim) return fail(h, ADG_ERR_INVALID, "axis out of range");
  std::string e;
  return wrap(h, adg::face_points(g, axis, n, q_minus, q_plus, d_low, d_high,
                                  (cudaStream_t)stream, &e), e);
}

int adg_riemann_points(adg_handle* h, const adg_grid* g, int64_t n, const double* normal,
                       int mode, const double* q_minus, const double* q_plus, double* out_a,
                       double* out_b, double* bpath, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (mode == 2 && is_el(g))
    return fail(h, ADG_ERR_UNSUPPORTED, "adg_riemann_points: speed mode for Euler and advection");
  if (!normal || n < 0 || mode < -1 || mode > 2 || (n > 0 && (!q_minus || !q_plus)) ||
      (mode >= 0 && !out_a) || (mode == 1 && !out_b))
    return fail(h, ADG_ERR_INVALID, "adg_riemann_points: bad arguments");
  std::string e;
  if (is_el(g))
    return wrap(h, adg::el_points(n, normal, mode, q_minus, q_plus, out_a, out_b, bpath,
                                  (cudaStream_t)stream, &e), e);
  if (mode < 0) return fail(h, ADG_ERR_INVALID, "path integral: nonconservative systems only");
  return wrap(h, adg::riemann_points(g, n, normal, mode, q_minus, q_plus, out_a, out_b,
                                     (cudaStream_t)stream, &e), e);
}

int adg_minmod(adg_handle* h, int64_t n, const double* a, const double* b, double* out,
               void* stream) {
  DeviceGuard dg(h);
  if (n < 0 || (n > 0 && (!a || !b || !out))) return fail(h, ADG_ERR_INVALID, "adg_minmod: bad arguments");
  std::string e;
  return wrap(h, adg::lim_minmod(a, b, n, out, (cudaStream_t)stream, &e), e);
}

int adg_relaxed_bounds(adg_handle* h, int dim, int nvars, const int64_t* cells, int nsub,
                       const double* padded_sub, double delta0, double eps, double* cmin_pad,
                       double* cmax_pad, double* lo_out, double* hi_out, void* stream) {
  DeviceGuard dg(h);
  if (dim < 1 || dim > 3 || nvars < 1 || !cells || nsub < 1 || !padded_sub || !cmin_pad ||
      !cmax_pad || !lo_out || !hi_out)
    return fail(h, ADG_ERR_INVALID, "adg_relaxed_bounds: bad arguments");
  std::string e;
  return wrap(h, adg::lim_relaxed_bounds(dim, nvars, cells, nsub, padded_sub, delta0, eps,
                                         cmin_pad, cmax_pad, lo_out, hi_out,
                                         (cudaStream_t)stream, &e), e);
}

int adg_detect_cells(adg_handle* h, const adg_grid* g, const double* cand,
                     const double* cand_sub, const double* lo, const double* hi,
                     uint8_t* troubled, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  if (!cand || !cand_sub || !lo || !hi || !troubled)
    return fail(h, ADG_ERR_INVALID, "adg_detect_cells: null array");
  std::string e;
  return wrap(h, adg::lim_detect_cells(g, cand, cand_sub, lo, hi, troubled,
                                       (cudaStream_t)stream, &e), e);
}

int adg_gather_windows(adg_handle* h, int dim, int nvars, const int64_t* padded_dims,
                       const double* padded, const int64_t* starts, int64_t nwin, int size,
                       double* out, void* stream) {
  DeviceGuard dg(h);
  if (dim < 1 || dim > 3 || nvars < 1 || !padded_dims || size < 1 || nwin < 0 ||
      (nwin > 0 && (!padded || !starts || !out)))
    return fail(h, ADG_ERR_INVALID, "adg_gather_windows: bad arguments");
  std::string e;
  return wrap(h, adg::lim_gather_windows(dim, nvars, padded_dims, padded, starts, nwin, size,
                                         out, (cudaStream_t)stream, &e), e);
}

int adg_volume_integral(adg_handle* h, const adg_grid* g, const double* q, const double* dt_dev,
                        double* vol_out, void* stream) {
  DeviceGuard dg(h);
  int rc = check_euler(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::volume_integral(g, q, dt_dev, vol_out, (cudaStream_t)stream, &e), e);
}

// linear, system-independent pieces: any number of quantities
static int check_linear(adg_handle* h, const adg_grid* g) {
  if (!g || g->dim < 1 || g->dim > 3 || g->degree < 0 || g->degree > 9 || g->nvars < 1)
    return fail(h, ADG_ERR_INVALID, "bad grid");
  for (int j = 0; j < g->dim; ++j)
    if (g->cells[j] < 0 || !(g->dx[j] > 0.0)) return fail(h, ADG_ERR_INVALID, "bad grid");
  if (!h->tables_loaded[g->degree])
    return fail(h, ADG_ERR_INVALID, "tables for this degree not uploaded (adg_set_tables)");
  return ADG_OK;
}

int adg_face_integral(adg_handle* h, const adg_grid* g, int axis, int side,
                      const double* d_values, const double* dt_dev, double* out, void* stream) {
  DeviceGuard dg(h);
  int rc = check_linear(h, g);
  if (rc) return rc;
  if (axis < 0 || axis >= g->dim || side < 0 || side > 1)
    return fail(h, ADG_ERR_INVALID, "axis / side out of range");
  std::string e;
  return wrap(h, adg::face_integral(g, axis, side, d_values, dt_dev, out, (cudaStream_t)stream,
                                    &e), e);
}

int adg_element_update(adg_handle* h, const adg_grid* g, const double* u, const double* vol,
                       const double* const* accs, int n_acc, double* u_out, void* stream) {
  DeviceGuard dg(h);
  int rc = check_linear(h, g);
  if (rc) return rc;
  if (n_acc < 0 || n_acc > 6 || (n_acc > 0 && !accs))
    return fail(h, ADG_ERR_INVALID, "0..6 face accumulators");
  std::string e;
  return wrap(h, adg::element_update(g, u, vol, accs, n_acc, u_out, (cudaStream_t)stream, &e), e);
}

int adg_muscl_windows(adg_handle* h, const adg_grid* g, const double* windows, int64_t n_windows,
                      const int32_t* count_dev, const double* dt_dev, double* avg_out,
                      uint8_t* failed, void* stream) {
  DeviceGuard dg(h);
  int rc = check_limiter(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::muscl_windows(g, windows, n_windows, count_dev, dt_dev, avg_out, failed,
                                    (cudaStream_t)stream, &e), e);
}

int adg_recover_subcells(adg_handle* h, const adg_grid* g, const double* ubar, double* u_out,
                         void* stream) {
  DeviceGuard dg(h);
  int rc = check_limiter(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::recover_subcells(g, ubar, u_out, (cudaStream_t)stream, &e), e);
}

int adg_flatten_cells(adg_handle* h, const adg_grid* g, double* nodal, const double* averages,
                      int32_t* nflat, void* stream) {
  DeviceGuard dg(h);
  int rc = check_limiter(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::flatten_cells(g, nodal, averages, nflat, (cudaStream_t)stream, &e), e);
}

int adg_flatten_ic(adg_handle* h, const adg_grid* g, double* u, int32_t* nflat, void* stream) {
  DeviceGuard dg(h);
  int rc = check_limiter(h, g);
  if (rc) return rc;
  std::string e;
  return wrap(h, adg::flatten_ic(g, u, nflat, (cudaStream_t)stream, &e), e);
}

int adg_comm_unique_id(void* id_out) {
  if (!id_out) return ADG_ERR_INVALID;
  std::string e;
  return adg::comm_unique_id(id_out, &e);
}

int adg_comm_init(adg_handle* h, const void* id, int nranks, int rank, adg_comm** out) {
  DeviceGuard dg(h);
  if (!h || !id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(h, ADG_ERR_INVALID, "adg_comm_init: bad arguments");
  *out = nullptr;
  std::string e;
  return wrap(h, adg::comm_init(h->device, id, nranks, rank, out, &e), e);
}

int adg_comm_destroy(adg_comm* c) { return adg::comm_destroy(c); }

static int check_comm(adg_handle* h, adg_comm* c) {
  if (!c) return fail(h, ADG_ERR_INVALID, "null communicator");
  if (adg::comm_device(c) != h->device)
    return fail(h, ADG_ERR_INVALID, "communicator and handle are bound to different devices");
  return ADG_OK;
}

int adg_halo_exchange(adg_handle* h, adg_comm* c, const adg_grid* g, const double* traces,
                      double* ghost_lo, double* ghost_hi, void* stream) {
  DeviceGuard dg(h);
  int rc = check_grid(h, g);
  if (rc) return rc;
  if ((rc = check_comm(h, c))) return rc;
  if (!traces || !ghost_lo || !ghost_hi)
    return fail(h, ADG_ERR_INVALID, "adg_halo_exchange: null buffer");
  std::string e;
  return wrap(h, adg::halo_exchange(c, g, traces, ghost_lo, ghost_hi, (cudaStream_t)stream, &e),
              e);
}

int adg_allreduce_reduce(adg_handle* h, adg_comm* c, adg_reduce* red, void* stream) {
  DeviceGuard dg(h);
  int rc = check_comm(h, c);
  if (rc) return rc;
  if (!red) return fail(h, ADG_ERR_INVALID, "adg_allreduce_reduce: null record");
  std::string e;
  return wrap(h, adg::allreduce_record(c, red, (cudaStream_t)stream, &e), e);
}

int adg_allreduce_sum(adg_handle* h, adg_comm* c, double* buf, int64_t n, void* stream) {
  DeviceGuard dg(h);
  int rc = check_comm(h, c);
  if (rc) return rc;
  if (n < 0 || (n > 0 && !buf)) return fail(h, ADG_ERR_INVALID, "adg_allreduce_sum: bad buffer");
  std::string e;
  return wrap(h, adg::allreduce_sum(c, buf, n, (cudaStream_t)stream, &e), e);
}

}  // extern "C"
