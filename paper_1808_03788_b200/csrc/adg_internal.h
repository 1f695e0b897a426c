// adg_internal.h -- host-side launchers shared between the .cu files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/aderdg_b200.h"

namespace adg {

// Per-device "done once" flag: kernel attributes (max dynamic shared memory,
// cluster sizes) are per device, so a process driving several devices sets
// them once on each (bit = device ordinal of the calling thread).
struct PerDevice {
  unsigned mask = 0;
  bool first() {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned bit = 1u << (d & 31);
    if (mask & bit) return false;
    mask |= bit;
    return true;
  }
};

constexpr int kReduceThreads = 256;
constexpr int64_t kReduceBlocksCap = 4096;  // fixed -> bitwise-reproducible totals
constexpr int64_t kUpdateBlocksCap = 148 * 8;

int64_t n_elements(const adg_grid* g);
int64_t reduce_blocks(const adg_grid* g);
int64_t update_blocks(const adg_grid* g);

size_t predict_workspace_bytes(int dim, int P, int num_sms, int64_t n_elem = 0);
int predict(const adg_grid* g, const double* u, const double* dt_dev, double tol, int max_iter,
            int min_iter, double* q_out, double* vol, double* traces, uint8_t* pred_bad,
            int32_t* sweeps, cudaStream_t st, int num_sms, double* ws, size_t ws_bytes,
            std::string* err, int64_t e_begin = 0, int64_t e_count = -1,
            const double* q_init = nullptr, int startup_only = 0);
// element ranges run on the shared-tile predictor only
bool predict_range_supported(const adg_grid* g);
bool predict_fold_supported(const adg_grid* g);

bool predict_stream_supported(const adg_grid* g);
size_t predict_stream_workspace_bytes(int P, int num_sms);
int predict_stream(const adg_grid* g, const double* u, const double* dt_dev, double tol,
                   int max_iter, int min_iter, double* q_out, double* vol, double* traces,
                   uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms, double* ws,
                   size_t ws_bytes, std::string* err);
// phase kernels over element batches for the 3-D N >= 7 tiles (adg_predictor_phased.cu)
bool predict_phased_supported(const adg_grid* g);
size_t predict_phased_workspace_bytes(int P, int64_t n_elem);
int predict_phased(const adg_grid* g, const double* u, const double* dt_dev, double tol,
                   int max_iter, int min_iter, double* q_out, double* vol, double* traces,
                   uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms, double* ws,
                   size_t ws_bytes, std::string* err);
// linear advection (adg_advection.cu)
int adv_predict(const adg_grid* g, const double* u, const double* dt_dev, double tol,
                int max_iter, int min_iter, double* q_out, double* vol, double* traces,
                uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms,
                std::string* err, const double* q_init = nullptr, int startup_only = 0);
int adv_spacetime_rate(const adg_grid* g, const double* q, double* rate, cudaStream_t st,
                       std::string* err);
int adv_face_flux(const adg_grid* g, int axis, const double* traces, const double* ghost_lo,
                  const double* ghost_hi, double* fd, cudaStream_t st, std::string* err);
int adv_update(const adg_grid* g, const double* u, const double* vol, const double* fd,
               const double* dt_dev, double* u_out, adg_reduce* red_next, double* partial,
               cudaStream_t st, std::string* err);
int adv_state_reduce(const adg_grid* g, const double* u, adg_reduce* red, double* partial,
                     cudaStream_t st, std::string* err);

// diffuse-interface elasticity, 2-D (adg_elasticity.cu)
int el_predict(const adg_grid* g, const double* u, const double* dt_dev, double tol,
               int max_iter, int min_iter, double* q_out, double* vol, double* traces,
               uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms,
               std::string* err);
int el_face_flux(const adg_grid* g, int axis, const double* traces, const double* ghost_lo,
                 const double* ghost_hi, double* fd, cudaStream_t st, std::string* err);
int el_update(const adg_grid* g, const double* u, const double* vol, const double* fd,
              const double* dt_dev, double* u_out, adg_reduce* red_next, double* partial,
              cudaStream_t st, std::string* err);
int el_state_reduce(const adg_grid* g, const double* u, adg_reduce* red, double* partial,
                    cudaStream_t st, std::string* err);

int state_reduce(const adg_grid* g, const double* u, adg_reduce* red, double* partial,
                 cudaStream_t st, std::string* err);
int timestep(const adg_grid* g, const adg_reduce* red, double cfl, const double* t_dev,
             double t_end, double* dt_dev, int32_t* status, cudaStream_t st, std::string* err);
int log_step(const double* row, int64_t ncols, const int32_t* status_in,
             const int32_t* elem_sweeps, int64_t n_elem, double* rows, int32_t* status,
             int32_t* sweeps, int64_t* cnt, cudaStream_t st, std::string* err);
int advance_time(double* t_dev, const double* dt_dev, double* t_out, cudaStream_t st,
                 std::string* err);
int face_flux(const adg_grid* g, int axis, const double* traces, const double* ghost_lo,
              const double* ghost_hi, double* dbar, cudaStream_t st, std::string* err);
int update(const adg_grid* g, const double* u, const double* vol, const double* fd,
           const double* dt_dev, double* u_out, adg_reduce* red_next, double* partial,
           cudaStream_t st, std::string* err);
int totals_finalize(const adg_grid* g, const double* partial, int64_t nblocks, double* out,
                    cudaStream_t st, std::string* err);

// limiter
int project_subcells(const adg_grid* g, const double* u, double* sub, double* cmin,
                     double* cmax, cudaStream_t st, std::string* err);
int detect(const adg_grid* g, const double* prev_sub, const double* cmin, const double* cmax,
           const double* cand, const uint8_t* pred_bad, double delta0, double eps,
           int force_all, const adg_subcell_ghosts* gh, uint8_t* troubled, int32_t* idx,
           int32_t* count, double* sub_out, double* cmin_out, double* cmax_out, cudaStream_t st,
           std::string* err);
int rescue(const adg_grid* g, const double* prev_sub, const int32_t* idx,
           const int32_t* count_dev, int32_t count_max, const double* dt_dev,
           const adg_subcell_ghosts* gh, double* u_out, int32_t* failed, double* sub_next,
           double* cmin_next, double* cmax_next, cudaStream_t st, std::string* err);
int flatten_ic(const adg_grid* g, double* u, int32_t* nflat, cudaStream_t st,
               std::string* err);

int muscl_windows(const adg_grid* g, const double* windows, int64_t nwin,
                  const int32_t* count_dev, const double* dt_dev, double* avg_out,
                  uint8_t* fail_each, cudaStream_t st, std::string* err);
int recover_subcells(const adg_grid* g, const double* ubar, double* out, cudaStream_t st,
                     std::string* err);
int flatten_cells(const adg_grid* g, double* nodal, const double* averages, int32_t* nflat,
                  cudaStream_t st, std::string* err);

// corrector module pieces (adg_pieces.cu)
int face_points(const adg_grid* g, int axis, int64_t n, const double* qm, const double* qp,
                double* dlow, double* dhigh, cudaStream_t st, std::string* err);
int volume_integral(const adg_grid* g, const double* q, const double* dt_dev, double* vol,
                    cudaStream_t st, std::string* err);
int face_integral(const adg_grid* g, int axis, int side, const double* d_values,
                  const double* dt_dev, double* out, cudaStream_t st, std::string* err);
int riemann_points(const adg_grid* g, int64_t n, const double* normal, int mode,
                   const double* qm, const double* qp, double* out_a, double* out_b,
                   cudaStream_t st, std::string* err);
int el_points(int64_t n, const double* normal, int mode, const double* qm, const double* qp,
              double* out_a, double* out_b, double* bpath, cudaStream_t st, std::string* err);
int extract_traces(const adg_grid* g, const double* q, double* out, cudaStream_t st,
                   std::string* err);
int spacetime_rate(const adg_grid* g, const double* q, double* rate, cudaStream_t st,
                   std::string* err);
int element_update(const adg_grid* g, const double* u, const double* vol,
                   const double* const* accs, int nacc, double* out, cudaStream_t st,
                   std::string* err);

// limiter module pieces (adg_pieces.cu)
int lim_minmod(const double* a, const double* b, int64_t n, double* out, cudaStream_t st,
               std::string* err);
int lim_relaxed_bounds(int dim, int m, const int64_t* cells, int nsub, const double* padded_sub,
                       double delta0, double eps, double* cmin_pad, double* cmax_pad, double* lo,
                       double* hi, cudaStream_t st, std::string* err);
int lim_detect_cells(const adg_grid* g, const double* cand, const double* sub, const double* lo,
                     const double* hi, uint8_t* out, cudaStream_t st, std::string* err);
int lim_gather_windows(int dim, int m, const int64_t* dims, const double* padded,
                       const int64_t* starts, int64_t nwin, int size, double* out,
                       cudaStream_t st, std::string* err);

void upload_tables(int degree, const double* blob, int64_t n, std::string* err, int* rc);

// multi-GPU exchange (adg_comm.cu, NCCL)
int comm_unique_id(void* out, std::string* err);
int comm_init(int device, const void* uid, int nranks, int rank, adg_comm** out,
              std::string* err);
int comm_destroy(adg_comm* c);
int comm_device(const adg_comm* c);
int halo_exchange(adg_comm* c, const adg_grid* g, const double* traces, double* ghost_lo,
                  double* ghost_hi, cudaStream_t st, std::string* err);
int allreduce_record(adg_comm* c, adg_reduce* red, cudaStream_t st, std::string* err);
int allreduce_sum(adg_comm* c, double* buf, int64_t n, cudaStream_t st, std::string* err);

}  // namespace adg
