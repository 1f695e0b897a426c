// adg_corrector.cu -- CFL reduction, Rusanov face coupling and the element
// update with a fused next-step wave-speed / conserved-total epilogue.
//
// References: corrector.compute_timestep (corrector.py:30-55),
// driver._face_states/_ghost_trace (driver.py:234-261),
// corrector.face_fluxes (corrector.py:100-129), face_integral
// (corrector.py:180-196), element_update (corrector.py:199-205),
// Simulation.conserved_totals (driver.py:344-350).
#include <algorithm>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

int64_t n_elements(const adg_grid* g) {
  int64_t n = 1;
  for (int j = 0; j < g->dim; ++j) n *= g->cells[j];
  return n;
}

int64_t reduce_blocks(const adg_grid* g) {
  const int64_t P = g->degree + 1;
  int64_t pd = 1;
  for (int j = 0; j < g->dim; ++j) pd *= P;
  const int64_t work = n_elements(g) * pd;
  return std::max<int64_t>(1, std::min<int64_t>((work + kReduceThreads - 1) / kReduceThreads,
                                                kReduceBlocksCap));
}

// blocks (= totals partials) of one update launch: persistent blocks over
// chunks of EB elements, EB = max(1, 768 / (P^d m)) as in UpdCfg (a fixed
// count keeps the global atomics few and the totals bitwise reproducible);
// never fewer than the reduction kernels use, so one partial buffer serves both
int64_t update_blocks(const adg_grid* g) {
  const int64_t P = g->degree + 1;
  int64_t pd = 1;
  for (int j = 0; j < g->dim; ++j) pd *= P;
  const int64_t eb = std::max<int64_t>(1, 256 / pd) * 2;   // >= UpdCfg::EB
  const int64_t nb = std::min<int64_t>(std::max<int64_t>(n_elements(g) / eb, 1), kUpdateBlocksCap);
  return std::max<int64_t>(nb, reduce_blocks(g));
}

// -------------------------------------------------------------------------
// Block-level fold of per-thread wave speeds / counts / totals.  Max is
// order independent; totals use a fixed shuffle tree + fixed warp order, so
// results are bitwise reproducible for a given grid.
template <int D>
__device__ void block_fold(double lam[3], unsigned nadm, unsigned nnf, const double* tot,
                           adg_reduce* red, double* partial) {
  constexpr int M = D + 2;
  constexpr int NW = kReduceThreads / 32;
  __shared__ double s_lam[NW][3];
  __shared__ unsigned s_cnt[NW][2];
  __shared__ double s_tot[NW][M];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int j = 0; j < D; ++j) lam[j] = fmax(lam[j], __shfl_xor_sync(0xffffffffu, lam[j], o));
  }
  nadm = __reduce_add_sync(0xffffffffu, nadm);
  nnf = __reduce_add_sync(0xffffffffu, nnf);
  double t[M];
  if (partial) {
#pragma unroll
    for (int v = 0; v < M; ++v) {
      t[v] = tot[v];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t[v] += __shfl_xor_sync(0xffffffffu, t[v], o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < D; ++j) s_lam[warp][j] = lam[j];
    s_cnt[warp][0] = nadm;
    s_cnt[warp][1] = nnf;
    if (partial) {
#pragma unroll
      for (int v = 0; v < M; ++v) s_tot[warp][v] = t[v];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double L[3] = {0.0, 0.0, 0.0};
    unsigned long long na = 0, nn = 0;
    double T[M];
#pragma unroll
    for (int v = 0; v < M; ++v) T[v] = 0.0;
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int j = 0; j < D; ++j) L[j] = fmax(L[j], s_lam[w][j]);
      na += s_cnt[w][0];
      nn += s_cnt[w][1];
      if (partial) {
#pragma unroll
        for (int v = 0; v < M; ++v) T[v] += s_tot[w][v];
      }
    }
    if (red) {
#pragma unroll
      for (int j = 0; j < D; ++j) atomic_max_pos(&red->lam_bits[j], L[j]);
      if (na) atomicAdd(reinterpret_cast<unsigned long long*>(&red->n_admissible), na);
      if (nn) atomicAdd(reinterpret_cast<unsigned long long*>(&red->n_nonfinite), nn);
    }
    if (partial) {
#pragma unroll
      for (int v = 0; v < M; ++v) partial[(size_t)blockIdx.x * M + v] = T[v];
    }
  }
}

// Per-node contribution to the fold: wave speeds over admissible nodes
// (corrector.py:42-52), non-finite detection (driver.py:197), weighted
// totals (driver.py:347-350 without the cell volume).
template <int D>
__device__ __forceinline__ void node_fold(const double* q, double gamma, double gm1, double wnode,
                                          double lam[3], unsigned& nadm, unsigned& nnf,
                                          double* tot) {
  constexpr int M = D + 2;
  bool fin = true;
#pragma unroll
  for (int v = 0; v < M; ++v) fin = fin && isfinite(q[v]);
  nnf += fin ? 0u : 1u;
  // admissibility (systems.py:225-229, exact verdict: the reference's IEEE
  // division decides within 1e-12 of cancellation) and the d wave speeds
  // |v_j| + c (systems.py:173-178) from ONE Newton-refined reciprocal of rho
  // (within a few ulp of the reference's quotients: dt to ~1e-16 relative)
  // instead of 2 d + 1 divisions: the update kernel is FP64-bound once the
  // folded state halves its HBM traffic
  if (fin && q[0] > 0.0) {
    const double r = rcp_nr(q[0]);
    double kin = q[1] * q[1];
#pragma unroll
    for (int j = 1; j < D; ++j) kin = kin + q[1 + j] * q[1 + j];
    const double x = 0.5 * kin * r;
    const double dd = q[D + 1] - x;
    const bool ppos = fabs(dd) > 1e-12 * (fabs(q[D + 1]) + fabs(x)) ? dd > 0.0
                                                                       : pressure<D>(q, gm1) > 0.0;
    if (ppos) {
      ++nadm;
      const double c = sqrt(gamma * (gm1 * dd) * r);
#pragma unroll
      for (int j = 0; j < D; ++j) lam[j] = fmax(lam[j], fabs(q[1 + j] * r) + c);
    }
  }
  if (tot) {
#pragma unroll
    for (int v = 0; v < M; ++v) tot[v] = fma(q[v], wnode, tot[v]);
  }
}

template <int D, int P>
__device__ __forceinline__ double node_weight(int node) {
  const DegreeTables& T = tab<P>();
  if (D == 1) return T.weights[node];
  if (D == 2) return T.weights[node / P] * T.weights[node % P];
  return T.weights[node / (P * P)] * T.weights[(node / P) % P] * T.weights[node % P];
}

template <int D, int P>
__global__ void __launch_bounds__(kReduceThreads)
state_reduce_kernel(const double* __restrict__ u, int64_t nodes, double gamma,
                    adg_reduce* red, double* partial) {
  constexpr int M = D + 2;
  constexpr int PD = ipow(P, D);
  const double gm1 = gamma - 1.0;
  double lam[3] = {0.0, 0.0, 0.0};
  unsigned nadm = 0, nnf = 0;
  double tot[M];
#pragma unroll
  for (int v = 0; v < M; ++v) tot[v] = 0.0;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    double q[M];
#pragma unroll
    for (int v = 0; v < M; ++v) q[v] = u[n * M + v];
    node_fold<D>(q, gamma, gm1, node_weight<D, P>((int)(n % PD)), lam, nadm, nnf,
                 partial ? tot : nullptr);
  }
  block_fold<D>(lam, nadm, nnf, tot, red, partial);
}

__global__ void zero_reduce_kernel(adg_reduce* red) {
  if (threadIdx.x < sizeof(adg_reduce) / 8)
    reinterpret_cast<unsigned long long*>(red)[threadIdx.x] = 0ull;
}

// corrector.py:47-55 plus the t_end clamp of driver.py:195
__global__ void timestep_kernel(const adg_reduce* red, int dim, double dx0, double dx1,
                                double dx2, double cfl, const double* t_dev, double t_end,
                                double* dt_out, int32_t* status) {
  const double dxs[3] = {dx0, dx1, dx2};
  int st = 0;
  if (red->n_admissible == 0) st |= ADG_STATUS_NO_ADMISSIBLE;
  if (red->n_nonfinite != 0) st |= ADG_STATUS_NONFINITE;
  double denom = 0.0;
  for (int j = 0; j < dim; ++j) denom += __longlong_as_double((long long)red->lam_bits[j]) / dxs[j];
  double dt = denom == 0.0 ? __longlong_as_double(0x7ff0000000000000LL) : cfl / denom;
  const double t = t_dev ? *t_dev : 0.0;
  const double rem = t_end - t;
  if (rem < dt) dt = rem;
  *dt_out = dt;
  if (status) *status |= st;
}

// batch history row (adg_log_step): max element sweep count (warp trees,
// warps in order), then the slot *cnt of the row / status / sweep logs
__global__ void __launch_bounds__(256)
log_step_kernel(const double* __restrict__ row, int64_t ncols, const int32_t* status_in,
                const int32_t* __restrict__ elem_sweeps, int64_t n_elem, double* rows,
                int32_t* status, int32_t* sweeps, int64_t* cnt) {
  __shared__ int s_max[8];
  int m = 0;
  for (int64_t e = threadIdx.x; e < n_elem; e += 256) m = max(m, elem_sweeps[e]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = m;
  __syncthreads();
  const int64_t c = *cnt;
  for (int64_t j = threadIdx.x; j < ncols; j += 256) rows[c * ncols + j] = row[j];
  if (threadIdx.x == 0) {
    int mm = s_max[0];
    for (int w = 1; w < 8; ++w) mm = max(mm, s_max[w]);
    sweeps[c] = mm;
    status[c] = *status_in;
  }
  __syncthreads();   // every thread has read *cnt
  if (threadIdx.x == 0) *cnt = c + 1;
}

__global__ void advance_time_kernel(double* t, const double* dt, double* t_out) {
  const double tn = *t + *dt;
  *t = tn;
  if (t_out) *t_out = tn;
}

// -------------------------------------------------------------------------
// Face coupling, streamed with TMA bulk copies.  A persistent block walks
// chunks of FB consecutive faces of one axis; for every face the minus-side
// and plus-side trace blocks (one element block each, padded to a 16-byte
// multiple) are fetched by lanes of warp 0 with cp.async.bulk into a
// double-buffered stage, and a thread per (face, tangential node) integrates
// sum_t w_t d_low(t) (corrector.py:100-129, :186) from shared memory.  The
// result is written element-major for both adjacent elements (coalesced).
// Face states follow driver._face_states/_ghost_trace (driver.py:234-261):
// periodic wrap, outflow copy, wall reflection, or caller ghost traces.
template <int D, int P>
struct FaceCfg {
  static constexpr int M = D + 2;
  static constexpr int PD = ipow(P, D);
  static constexpr int PF = PD / P;                  // tangential nodes per face
  static constexpr int TB = PD * M + ((PD * M) & 1); // trace element block (doubles)
  static constexpr int FB = (128 / PF) > 0 ? (128 / PF) : 1;
  static constexpr int NT = ((FB * PF + 31) / 32) * 32 < 64 ? 64 : ((FB * PF + 31) / 32) * 32;
  static constexpr int STAGE = 2 * FB * TB;
  // one stage per block: the kernel is latency bound, so four resident
  // blocks (16 warps) per SM beat in-block double buffering
  static constexpr int NSTAGE = 1;
  static constexpr size_t SMEM = (size_t)NSTAGE * STAGE * 8;
};

template <int D, int P, int AX>
__global__ void __launch_bounds__(FaceCfg<D, P>::NT)
face_kernel(const double* __restrict__ traces, const double* __restrict__ ghost_lo,
            const double* __restrict__ ghost_hi, double* __restrict__ fd, int64_t c0,
            int64_t c1, int64_t c2, int bc_lo, int bc_hi, double gamma) {
  using C = FaceCfg<D, P>;
  constexpr int axis = AX;
  constexpr int M = C::M, PF = C::PF, TB = C::TB, FB = C::FB, STAGE = C::STAGE;
  extern __shared__ __align__(128) double fsm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int s_ref[2][FB][2];           // wall reflection of minus / plus state
  __shared__ int64_t s_dst[2][FB][2];       // element receiving the face as high / low face
  const DegreeTables& T = tab<P>();
  const double gm1 = gamma - 1.0;
  const int tid = threadIdx.x;
  const int64_t n[3] = {c0, c1, c2};
  int64_t nf[3] = {c0, c1, c2};
  nf[axis] += 1;
  const int64_t faces = nf[0] * (D >= 2 ? nf[1] : 1) * (D == 3 ? nf[2] : 1);
  const int64_t E = n[0] * (D >= 2 ? n[1] : 1) * (D == 3 ? n[2] : 1);
  const size_t fstride = (size_t)E * TB;
  const double* tr_lo = traces + (size_t)(2 * axis) * fstride;
  const double* tr_hi = tr_lo + fstride;
  const int64_t nchunks = (faces + FB - 1) / FB;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // warp 0: lane 2f + side fetches the minus (side 0) / plus (side 1) state
  // block of face f of chunk c into stage stg
  auto issue = [&](int stg, int64_t c) {
    const int64_t f0 = c * FB;
    const int nfb = (int)((faces - f0) < FB ? (faces - f0) : FB);
    if (tid == 0) mbar_expect_tx(&bar[stg], (uint32_t)(2 * nfb * TB * 8));
    __syncwarp();
    for (int lane = tid; lane < 2 * nfb; lane += 32) {
      const int f = lane >> 1, side = lane & 1;
      int64_t cc[3] = {0, 0, 0};
      int64_t r = f0 + f;
      for (int j = D - 1; j >= 0; --j) {
        cc[j] = r % nf[j];
        r /= nf[j];
      }
      const int64_t ca = cc[axis];
      auto elem = [&](int64_t caxis) {
        int64_t e = 0;
        for (int j = 0; j < D; ++j) e = e * n[j] + (j == axis ? caxis : cc[j]);
        return e;
      };
      int64_t plane = 0;
      for (int j = 0; j < D; ++j)
        if (j != axis) plane = plane * n[j] + cc[j];
      const double* src;
      int refl = 0;
      if (side == 0) {   // minus state: high trace of the low-side element
        if (ca == 0) {
          if (bc_lo == ADG_BC_PERIODIC) src = tr_hi + (size_t)elem(n[axis] - 1) * TB;
          else if (bc_lo == ADG_BC_GHOST) src = ghost_lo + (size_t)plane * TB;
          else { src = tr_lo + (size_t)elem(0) * TB; refl = bc_lo == ADG_BC_WALL; }
        } else {
          src = tr_hi + (size_t)elem(ca - 1) * TB;
        }
        s_dst[stg][f][0] = ca >= 1 ? elem(ca - 1) : -1;
      } else {           // plus state: low trace of the high-side element
        if (ca == n[axis]) {
          if (bc_hi == ADG_BC_PERIODIC) src = tr_lo + (size_t)elem(0) * TB;
          else if (bc_hi == ADG_BC_GHOST) src = ghost_hi + (size_t)plane * TB;
          else { src = tr_hi + (size_t)elem(n[axis] - 1) * TB; refl = bc_hi == ADG_BC_WALL; }
        } else {
          src = tr_lo + (size_t)elem(ca) * TB;
        }
        s_dst[stg][f][1] = ca < n[axis] ? elem(ca) : -1;
      }
      s_ref[stg][f][side] = refl;
      bulk_g2s(fsm + stg * STAGE + (size_t)lane * TB, src, TB * 8, &bar[stg]);
    }
  };

  uint32_t phase[2] = {0u, 0u};
  int64_t c = blockIdx.x;
  if (tid < 32 && c < nchunks) issue(0, c);
  __syncthreads();
  // element-face trace blocks are written by the predictor's owner roles:
  // x faces [j][k][t], y faces [k][t][i], z faces [t][i][j] (2-D: x [j][t],
  // y [t][i]); (ta, tb) are the ascending tangential indices
  constexpr int SA = D == 3 ? (AX == 0 ? P * P : (AX == 1 ? 1 : P)) : (D == 2 ? (AX == 0 ? P : 1) : 0);
  constexpr int SB = D == 3 ? (AX == 0 ? P : (AX == 1 ? P * P : 1)) : 0;
  constexpr int ST = D == 3 ? (AX == 0 ? 1 : (AX == 1 ? P : P * P)) : (D == 2 ? (AX == 0 ? 1 : P) : 1);
  for (int i = 0; c < nchunks; ++i, c += gridDim.x) {
    const int stg = C::NSTAGE == 2 ? (i & 1) : 0;
    const int64_t cn = c + gridDim.x;
    if (C::NSTAGE == 2 && tid < 32 && cn < nchunks) issue(stg ^ 1, cn);
    if (C::NSTAGE == 1 && i > 0) {
      if (tid < 32) issue(0, c);
      __syncthreads();
    }
    mbar_wait(&bar[stg], phase[stg]);
    phase[stg] ^= 1u;
    const int64_t f0 = c * FB;
    const int nfb = (int)((faces - f0) < FB ? (faces - f0) : FB);
    if (tid < nfb * PF) {
      const int f = tid / PF, tg = tid - f * PF;
      const int ta = D == 3 ? tg / P : tg;
      const int tb = D == 3 ? tg % P : 0;
      const int base = ta * SA + tb * SB;
      const double* pm = fsm + stg * STAGE + (size_t)(2 * f) * TB + base * M;
      const double* pp = pm + TB;
      const bool rm = s_ref[stg][f][0], rp = s_ref[stg][f][1];
      double acc[M];
#pragma unroll
      for (int v = 0; v < M; ++v) acc[v] = 0.0;
#pragma unroll
      for (int t = 0; t < P; ++t) {
        double qm[M], qp[M];
#pragma unroll
        for (int v = 0; v < M; ++v) {
          qm[v] = pm[t * ST * M + v];
          qp[v] = pp[t * ST * M + v];
        }
        if (rm) qm[1 + axis] = -qm[1 + axis];   // systems.py:231-234
        if (rp) qp[1 + axis] = -qp[1 + axis];
        double fm[M], fp[M];
        const double s = nan_max(flux_eig_axis<D>(qm, gamma, gm1, axis, fm),
                              flux_eig_axis<D>(qp, gamma, gm1, axis, fp));
        const double hs = 0.5 * s;
        const double wt = T.weights[t];
#pragma unroll
        for (int v = 0; v < M; ++v) {
          const double central = 0.5 * (fm[v] + fp[v]);
          const double dlow = (central + 0.0) - hs * (qp[v] - qm[v]);
          acc[v] = fma(wt, dlow, acc[v]);
        }
      }
      // element-major face terms fd[E][D][2 sides][P^(d-1)][m]: the face is
      // the high face of its low-side element and the low face of its
      // high-side element (periodic: face n_a repeats face 0)
      constexpr size_t FBLK = (size_t)PF * M;
      const int64_t eL = s_dst[stg][f][0], eR = s_dst[stg][f][1];
      if (eL >= 0) {
        double* o = fd + ((size_t)eL * (2 * D) + 2 * axis + 1) * FBLK + (size_t)tg * M;
#pragma unroll
        for (int v = 0; v < M; ++v) o[v] = acc[v];
      }
      if (eR >= 0) {
        double* o = fd + ((size_t)eR * (2 * D) + 2 * axis) * FBLK + (size_t)tg * M;
#pragma unroll
        for (int v = 0; v < M; ++v) o[v] = acc[v];
      }
    }
    __syncthreads();   // stage and face metadata free for the next prefetch
  }
}

// -------------------------------------------------------------------------
// Element update, streamed with TMA bulk copies.  Each persistent block walks
// chunks of EB consecutive elements; a chunk is three contiguous, 16-byte
// aligned blocks (u, vol, element-major face terms) fetched by one elected
// thread with cp.async.bulk into a double-buffered stage (the next chunk
// lands while the current one is computed), a thread per node forms
// u + (vol - sum of face integrals) / mass in the reference's order
// (corrector.py:180-205) in place, folds the new state into the next step's
// wave-speed record and the conserved-total partial, and the chunk leaves
// through one bulk store.  A ragged tail chunk uses plain loads/stores.
template <int D, int P>
struct UpdCfg {
  static constexpr int M = D + 2;
  static constexpr int PD = ipow(P, D);
  static constexpr int PF = PD / P;
  static constexpr int FE = 2 * D * PF * M;            // face-term values per element
  static constexpr int EB0 = (256 / PD) > 0 ? (256 / PD) : 1;
  // chunk byte counts must be multiples of 16 for the bulk engine
  static constexpr int EB = ((EB0 * PD * M) % 2 == 0) ? EB0 : 2 * EB0;
  static constexpr int CU = EB * PD * M;               // state values per chunk
  static constexpr int CF = EB * FE;                   // face values per chunk
  static constexpr int STAGE = 2 * CU + CF;            // doubles per stage
  // double-buffered unless two stages exceed the shared-memory budget
  static constexpr int NSTAGE = (2 * STAGE * 8 <= 200 * 1024) ? 2 : 1;
  static constexpr size_t SMEM = (size_t)NSTAGE * STAGE * 8;
};

template <int D, int P>
__device__ __forceinline__ void update_chunk(const double* SU_in, const double* SV,
                                             const double* SF, double* SU_out, int neb,
                                             const double* s_w, const double* s_l,
                                             const double* s_r, double dt, double cv,
                                             const double* dx, double gamma, double gm1,
                                             double* lam, unsigned& nadm, unsigned& nnf,
                                             double* tot) {
  using C = UpdCfg<D, P>;
  constexpr int M = C::M, PD = C::PD, PF = C::PF, FE = C::FE;
  for (int y = threadIdx.x; y < neb * PD; y += kReduceThreads) {
    const int el = y / PD, node = y - el * PD;
    int k[3] = {0, 0, 0};
    if (D == 1) k[0] = node;
    if (D == 2) { k[0] = node / P; k[1] = node % P; }
    if (D == 3) { k[0] = node / (P * P); k[1] = (node / P) % P; k[2] = node % P; }
    double total[M];
#pragma unroll
    for (int v = 0; v < M; ++v) total[v] = SV ? SV[y * M + v] : 0.0;   // folded: SU_in holds u + vol / mass
#pragma unroll
    for (int a = 0; a < D; ++a) {
      int tg = 0;
      double wtan = 1.0;
      bool first = true;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j == a) continue;
        tg = tg * P + k[j];
        wtan = first ? s_w[k[j]] : wtan * s_w[k[j]];
        first = false;
      }
      const double sc = dt * (cv / dx[a]);
      const double* dlo = SF + el * FE + (2 * a) * PF * M + tg * M;
      const double* dhi = dlo + PF * M;
      const double vl = s_l[k[a]], vr = s_r[k[a]];
#pragma unroll
      for (int v = 0; v < M; ++v) {
        const double blo = (D > 1) ? (-dlo[v]) * wtan : -dlo[v];
        total[v] -= sc * (vl * blo);
      }
#pragma unroll
      for (int v = 0; v < M; ++v) {
        const double bhi = (D > 1) ? dhi[v] * wtan : dhi[v];
        total[v] -= sc * (vr * bhi);
      }
    }
    double wnode;
    if (D == 1) wnode = s_w[k[0]];
    else if (D == 2) wnode = s_w[k[0]] * s_w[k[1]];
    else wnode = s_w[k[0]] * s_w[k[1]] * s_w[k[2]];
    const double mass = cv * wnode;
    double q[M];
    if (SV) {
#pragma unroll
      for (int v = 0; v < M; ++v) q[v] = SU_in[y * M + v] + total[v] / mass;
    } else {
      // folded: the predictor already applied 1 / mass to the volume term
      // the same way (one reciprocal per node instead of m divisions)
      const double rmass = 1.0 / mass;
#pragma unroll
      for (int v = 0; v < M; ++v) q[v] = fma(total[v], rmass, SU_in[y * M + v]);
    }
#pragma unroll
    for (int v = 0; v < M; ++v) SU_out[y * M + v] = q[v];
    node_fold<D>(q, gamma, gm1, wnode, lam, nadm, nnf, tot);
  }
}

#ifndef ADG_UPD_MINB
#define ADG_UPD_MINB 3   // 80 registers: three CTAs per SM (C2 step 11.92 -> 11.87 ms)
#endif
template <int D, int P>
__global__ void __launch_bounds__(kReduceThreads, ADG_UPD_MINB)
update_kernel(const double* __restrict__ u, const double* __restrict__ vol,
              const double* __restrict__ fd, const double* __restrict__ dt_dev,
              double* __restrict__ u_out, int64_t E, double dx0, double dx1, double dx2,
              double gamma, adg_reduce* red, double* partial) {
  using C = UpdCfg<D, P>;
  constexpr int M = C::M, PD = C::PD, FE = C::FE, EB = C::EB, CU = C::CU, CF = C::CF;
  constexpr int STAGE = C::STAGE;
  extern __shared__ __align__(128) double usm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double s_w[P], s_l[P], s_r[P];
  const DegreeTables& T = tab<P>();
  const int tid = threadIdx.x;
  // The grid has one block per totals partial (never fewer than the
  // reduction kernels use); on small grids most blocks own no chunk: they
  // leave their zero partial and exit (what block_fold would write)
  if ((int64_t)blockIdx.x >= E / EB && !(blockIdx.x == 0 && E % EB)) {
    if (partial && tid < M) partial[(size_t)blockIdx.x * M + tid] = 0.0;
    return;
  }
  if (tid < P) {
    s_w[tid] = T.weights[tid];
    s_l[tid] = T.left[tid];
    s_r[tid] = T.right[tid];
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double gm1 = gamma - 1.0;
  const double dt = *dt_dev;
  const double dx[3] = {dx0, dx1, dx2};
  const double cv = dx0 * (D >= 2 ? dx1 : 1.0) * (D == 3 ? dx2 : 1.0);
  double lam[3] = {0.0, 0.0, 0.0};
  unsigned nadm = 0, nnf = 0;
  double tot[M];
#pragma unroll
  for (int v = 0; v < M; ++v) tot[v] = 0.0;
  double* tp = partial ? tot : nullptr;

  const int64_t nfull = E / EB;             // chunks served by the bulk engine
  auto issue = [&](int stg, int64_t c) {
    double* st = usm + stg * STAGE;
    const int64_t e0 = c * EB;
    mbar_expect_tx(&bar[stg], (uint32_t)((vol ? STAGE : STAGE - CU) * 8));
    bulk_g2s(st, u + (size_t)e0 * PD * M, CU * 8, &bar[stg]);
    if (vol) bulk_g2s(st + CU, vol + (size_t)e0 * PD * M, CU * 8, &bar[stg]);
    bulk_g2s(st + 2 * CU, fd + (size_t)e0 * FE, CF * 8, &bar[stg]);
  };
  uint32_t phase[2] = {0u, 0u};
  int64_t c = blockIdx.x;
  if (C::NSTAGE == 2 && tid == 0 && c < nfull) issue(0, c);
  for (int i = 0; c < nfull; ++i, c += gridDim.x) {
    const int stg = C::NSTAGE == 2 ? (i & 1) : 0;
    const int64_t cn = c + gridDim.x;
    if (tid == 0) {
      if (C::NSTAGE == 2) {
        if (cn < nfull) {
          bulk_wait_read_all();   // the other stage's bulk store has left smem
          issue(stg ^ 1, cn);
        }
      } else {
        bulk_wait_read_all();
        issue(0, c);
      }
    }
    mbar_wait(&bar[stg], phase[stg]);
    phase[stg] ^= 1u;
    double* st = usm + stg * STAGE;
    update_chunk<D, P>(st, vol ? st + CU : nullptr, st + 2 * CU, st, EB, s_w, s_l, s_r, dt, cv, dx,
                       gamma, gm1, lam, nadm, nnf, tp);
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      bulk_s2g(u_out + (size_t)c * EB * PD * M, st, CU * 8);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_all();
  __syncthreads();
  // ragged tail (E % EB elements) with plain loads / stores, by block 0
  const int tail = (int)(E - nfull * EB);
  if (tail > 0 && blockIdx.x == 0) {
    double* st = usm;
    const size_t off = (size_t)nfull * EB * PD * M;
    for (int x = tid; x < tail * PD * M; x += kReduceThreads) {
      st[x] = u[off + x];
      if (vol) st[CU + x] = vol[off + x];
    }
    for (int x = tid; x < tail * FE; x += kReduceThreads)
      st[2 * CU + x] = fd[(size_t)nfull * EB * FE + x];
    __syncthreads();
    update_chunk<D, P>(st, vol ? st + CU : nullptr, st + 2 * CU, st, tail, s_w, s_l, s_r, dt, cv,
                       dx, gamma, gm1, lam, nadm, nnf, tp);
    __syncthreads();
    for (int x = tid; x < tail * PD * M; x += kReduceThreads) u_out[off + x] = st[x];
  }
  block_fold<D>(lam, nadm, nnf, tot, red, partial);
}

template <int M>
__global__ void totals_finalize_kernel(const double* __restrict__ partial, int64_t nb, double cv,
                                       double* out) {
  // 1024 threads: fixed strided partial sums, then a fixed shared-memory
  // tree -> bitwise reproducible for a given partial count
  __shared__ double sm[1024];
  const int t = threadIdx.x;
  for (int v = 0; v < M; ++v) {
    double s = 0.0;
    for (int64_t b = t; b < nb; b += 1024) s += partial[b * M + v];
    sm[t] = s;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
      if (t < o) sm[t] += sm[t + o];
      __syncthreads();
    }
    if (t == 0) out[v] = cv * sm[0];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ launchers
#define ADG_SWITCH_DP(FN, ...)                                                   \
  do {                                                                           \
    const int P_ = g->degree + 1;                                                \
    switch (g->dim * 16 + P_) {                                                  \
      case 16 + 1: FN<1, 1>(__VA_ARGS__); break;                                 \
      case 16 + 2: FN<1, 2>(__VA_ARGS__); break;                                 \
      case 16 + 3: FN<1, 3>(__VA_ARGS__); break;                                 \
      case 16 + 4: FN<1, 4>(__VA_ARGS__); break;                                 \
      case 16 + 5: FN<1, 5>(__VA_ARGS__); break;                                 \
      case 16 + 6: FN<1, 6>(__VA_ARGS__); break;                                 \
      case 16 + 7: FN<1, 7>(__VA_ARGS__); break;                                 \
      case 16 + 8: FN<1, 8>(__VA_ARGS__); break;                                 \
      case 16 + 9: FN<1, 9>(__VA_ARGS__); break;                                 \
      case 16 + 10: FN<1, 10>(__VA_ARGS__); break;                               \
      case 32 + 1: FN<2, 1>(__VA_ARGS__); break;                                 \
      case 32 + 2: FN<2, 2>(__VA_ARGS__); break;                                 \
      case 32 + 3: FN<2, 3>(__VA_ARGS__); break;                                 \
      case 32 + 4: FN<2, 4>(__VA_ARGS__); break;                                 \
      case 32 + 5: FN<2, 5>(__VA_ARGS__); break;                                 \
      case 32 + 6: FN<2, 6>(__VA_ARGS__); break;                                 \
      case 32 + 7: FN<2, 7>(__VA_ARGS__); break;                                 \
      case 32 + 8: FN<2, 8>(__VA_ARGS__); break;                                 \
      case 32 + 9: FN<2, 9>(__VA_ARGS__); break;                                 \
      case 32 + 10: FN<2, 10>(__VA_ARGS__); break;                               \
      case 48 + 1: FN<3, 1>(__VA_ARGS__); break;                                 \
      case 48 + 2: FN<3, 2>(__VA_ARGS__); break;                                 \
      case 48 + 3: FN<3, 3>(__VA_ARGS__); break;                                 \
      case 48 + 4: FN<3, 4>(__VA_ARGS__); break;                                 \
      case 48 + 5: FN<3, 5>(__VA_ARGS__); break;                                 \
      case 48 + 6: FN<3, 6>(__VA_ARGS__); break;                                 \
      case 48 + 7: FN<3, 7>(__VA_ARGS__); break;                                 \
      case 48 + 8: FN<3, 8>(__VA_ARGS__); break;                                 \
      case 48 + 9: FN<3, 9>(__VA_ARGS__); break;                                 \
      case 48 + 10: FN<3, 10>(__VA_ARGS__); break;                               \
      default: *err = "unsupported dim/degree"; return ADG_ERR_UNSUPPORTED;      \
    }                                                                            \
  } while (0)

static int check_launch(std::string* err) {
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

template <int D, int P>
static void launch_state_reduce(const adg_grid* g, const double* u, adg_reduce* red,
                                double* partial, cudaStream_t st) {
  const int64_t nodes = n_elements(g) * ipow(P, D);
  state_reduce_kernel<D, P><<<(unsigned)reduce_blocks(g), kReduceThreads, 0, st>>>(
      u, nodes, g->gamma, red, partial);
}

int state_reduce(const adg_grid* g, const double* u, adg_reduce* red, double* partial,
                 cudaStream_t st, std::string* err) {
  if (red) zero_reduce_kernel<<<1, 32, 0, st>>>(red);
  ADG_SWITCH_DP(launch_state_reduce, g, u, red, partial, st);
  return check_launch(err);
}

int timestep(const adg_grid* g, const adg_reduce* red, double cfl, const double* t_dev,
             double t_end, double* dt_dev, int32_t* status, cudaStream_t st, std::string* err) {
  timestep_kernel<<<1, 1, 0, st>>>(red, g->dim, g->dx[0], g->dx[1], g->dx[2], cfl, t_dev, t_end,
                                   dt_dev, status);
  return check_launch(err);
}

int advance_time(double* t_dev, const double* dt_dev, double* t_out, cudaStream_t st,
                 std::string* err) {
  advance_time_kernel<<<1, 1, 0, st>>>(t_dev, dt_dev, t_out);
  return check_launch(err);
}

int log_step(const double* row, int64_t ncols, const int32_t* status_in,
             const int32_t* elem_sweeps, int64_t n_elem, double* rows, int32_t* status,
             int32_t* sweeps, int64_t* cnt, cudaStream_t st, std::string* err) {
  log_step_kernel<<<1, 256, 0, st>>>(row, ncols, status_in, elem_sweeps, n_elem, rows, status,
                                     sweeps, cnt);
  return check_launch(err);
}

template <int D, int P>
static void launch_face(const adg_grid* g, int axis, const double* traces, const double* glo,
                        const double* ghi, double* fd, cudaStream_t st) {
  using C = FaceCfg<D, P>;
  int64_t nf[3] = {g->cells[0], g->cells[1], g->cells[2]};
  nf[axis] += 1;
  int64_t faces = 1;
  for (int j = 0; j < D; ++j) faces *= nf[j];
  const int64_t chunks = (faces + C::FB - 1) / C::FB;
  auto kern = axis == 0 ? face_kernel<D, P, 0>
                        : (axis == 1 ? face_kernel<D, P, (D > 1 ? 1 : 0)>
                                     : face_kernel<D, P, (D > 2 ? 2 : 0)>);
  static PerDevice attr[3];
  if (attr[axis].first())
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  const int64_t blocks = std::min<int64_t>(chunks, 148 * 8);
  kern<<<(unsigned)blocks, C::NT, C::SMEM, st>>>(
      traces, glo, ghi, fd, g->cells[0], D >= 2 ? g->cells[1] : 1, D == 3 ? g->cells[2] : 1,
      g->bc[axis][0], g->bc[axis][1], g->gamma);
}

int face_flux(const adg_grid* g, int axis, const double* traces, const double* ghost_lo,
              const double* ghost_hi, double* dbar, cudaStream_t st, std::string* err) {
  if (axis < 0 || axis >= g->dim) {
    *err = "axis out of range";
    return ADG_ERR_INVALID;
  }
  if ((g->bc[axis][0] == ADG_BC_GHOST && !ghost_lo) ||
      (g->bc[axis][1] == ADG_BC_GHOST && !ghost_hi)) {
    *err = "ghost boundary without ghost traces";
    return ADG_ERR_INVALID;
  }
  ADG_SWITCH_DP(launch_face, g, axis, traces, ghost_lo, ghost_hi, dbar, st);
  return check_launch(err);
}

template <int D, int P>
static void launch_update(const adg_grid* g, const double* u, const double* vol, const double* fd,
                          const double* dt_dev, double* u_out, adg_reduce* red, double* partial,
                          cudaStream_t st) {
  static PerDevice attr;
  if (attr.first())
    cudaFuncSetAttribute(update_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)UpdCfg<D, P>::SMEM);
  update_kernel<D, P><<<(unsigned)update_blocks(g), kReduceThreads, UpdCfg<D, P>::SMEM, st>>>(
      u, vol, fd, dt_dev, u_out, n_elements(g), g->dx[0], D >= 2 ? g->dx[1] : 1.0,
      D == 3 ? g->dx[2] : 1.0, g->gamma, red, partial);
}

int update(const adg_grid* g, const double* u, const double* vol, const double* fd,
           const double* dt_dev, double* u_out, adg_reduce* red_next, double* partial,
           cudaStream_t st, std::string* err) {
  if (!fd) {
    *err = "missing face data";
    return ADG_ERR_INVALID;
  }
  if (red_next) zero_reduce_kernel<<<1, 32, 0, st>>>(red_next);
  if (g->flags & ADG_GRID_FOLD_STATE) {
    // the predictor left w = u + vol / mass in `vol`: it takes u's place
    u = vol;
    vol = nullptr;
  }
  ADG_SWITCH_DP(launch_update, g, u, vol, fd, dt_dev, u_out, red_next, partial, st);
  return check_launch(err);
}

int totals_finalize(const adg_grid* g, const double* partial, int64_t nb, double* out,
                    cudaStream_t st, std::string* err) {
  double cv = 1.0;
  for (int j = 0; j < g->dim; ++j) cv *= g->dx[j];
  if (g->nvars == 1) {
    totals_finalize_kernel<1><<<1, 1024, 0, st>>>(partial, nb, cv, out);
    return check_launch(err);
  }
  if (g->nvars == 9) {   // elasticity-di
    totals_finalize_kernel<9><<<1, 1024, 0, st>>>(partial, nb, cv, out);
    return check_launch(err);
  }
  switch (g->dim) {
    case 1: totals_finalize_kernel<3><<<1, 1024, 0, st>>>(partial, nb, cv, out); break;
    case 2: totals_finalize_kernel<4><<<1, 1024, 0, st>>>(partial, nb, cv, out); break;
    case 3: totals_finalize_kernel<5><<<1, 1024, 0, st>>>(partial, nb, cv, out); break;
    default: *err = "bad dim"; return ADG_ERR_INVALID;
  }
  return check_launch(err);
}

}  // namespace adg
