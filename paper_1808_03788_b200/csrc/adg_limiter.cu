// adg_limiter.cu -- a posteriori subcell finite-volume limiter (sm_100a).
//
// References: driver._limit / _pad_subcells / _boundary_slab
// (driver.py:265-340), limiter.project_to_subcells (limiter.py:27-33),
// relaxed_bounds (:51-73), detect_troubled (:76-86), gather_windows
// (:89-101), muscl_subcell_step/_muscl_once (:104-202), minmod (:45-48),
// recover_from_subcells (:36-42), flatten_inadmissible (:205-223) and the
// IC flattening of Simulation.project_initial_condition (driver.py:137-152).
//
// Device layout: prev_sub[E][S^d][m] subcell averages of u^n (S = 2N+1),
// cmin/cmax[E][m] their per-cell extrema.  Ghost subcells outside the grid
// are never materialised: a global subcell coordinate is mapped through the
// face kind per axis (periodic wrap, outflow clamp, wall mirror + normal
// momentum flip), which reproduces the reference's sequential per-axis
// padding exactly, corners included.
//
// Troubled cells are compacted with an atomic counter; every rescue reads
// only t^n data and writes only its own cell, so the result does not depend
// on the compaction order.  One CTA rescues one cell (window, MUSCL-Hancock
// half step, Rusanov subcell faces, first-order retry, recovery, flatten).
#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

template <int D, int P, int SYS>
struct LimCfg {
  // SYS 0: CompressibleEuler (m = d + 2); SYS 1: LinearAdvection (m = 1)
  static constexpr int M = SYS == 1 ? 1 : D + 2;
  static constexpr int S = 2 * P - 1;
  static constexpr int PD = ipow(P, D);
  static constexpr int SD = ipow(S, D);
  static constexpr int W = S + 4;              // window edge
  static constexpr int WD = ipow(W, D);
  static constexpr int R = S + 2;              // 1-halo region edge
  static constexpr int RD = ipow(R, D);
  static constexpr int NT = 256;
};

struct LimGrid {
  int64_t n[3];
  int bc[3][2];
  double gm1, gamma;
  double h[3];  // subcell widths dx_j / S
  int prim;     // predictor_mode == "primitive": MUSCL-Hancock in primitive variables
  double a[3];  // LinearAdvection velocity (SYS 1)
  // ADG_BC_GHOST ("exact") faces: caller-evaluated exterior subcell slabs
  // (adg_subcell_ghosts); L = their layer count
  const double* slab[3][2];
  int L;
};

// ---------------------------------------------------------------- helpers
template <int D>
__device__ __forceinline__ int64_t cell_index(const int64_t* c, const int64_t* n) {
  int64_t e = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) e = e * n[j] + c[j];
  return e;
}


// ------------------------------------------------- system policy (SYS)
// The limiter's physics (limiter.py runs on any HyperbolicSystem):
// admissibility, directional flux, the subcell Rusanov pair and the
// primitive-mode conversions.  SYS 0 = CompressibleEuler (systems.py:112-234),
// SYS 1 = LinearAdvection (systems.py:77-109: admissible = finite, F_j = a_j q,
// |lambda| = |a_j|, reflect = identity, primitives = conserved).
template <int D, int SYS>
__device__ __forceinline__ bool lim_adm(const double* q, double gm1) {
  if constexpr (SYS == 1) return isfinite(q[0]);
  else return admissible<D>(q, gm1);
}
template <int D, int SYS>
__device__ __forceinline__ bool lim_adm_fast(const double* q, double gm1) {
  if constexpr (SYS == 1) return isfinite(q[0]);
  else return admissible_fast<D>(q, gm1);
}
template <int D, int SYS>
__device__ __forceinline__ void lim_flux(const double* q, const LimGrid& G, int j, double* f) {
  if constexpr (SYS == 1) f[0] = G.a[j] * q[0];
  else flux_axis<D>(q, G.gm1, j, f);
}
template <int D, int SYS>
__device__ __forceinline__ void lim_rusanov(const double* qm, const double* qp, int j,
                                            const LimGrid& G, double* dlow, double* dhigh) {
  if constexpr (SYS == 1) {
    // face_fluxes (corrector.py:100-129) with s = max(|a_j|, |a_j|)
    const double s = fabs(G.a[j]);
    const double central = 0.5 * (G.a[j] * qm[0] + G.a[j] * qp[0]);
    const double diss = (0.5 * s) * (qp[0] - qm[0]);
    dlow[0] = (central + 0.0) - diss;
    dhigh[0] = (-central + 0.0) + diss;
  } else {
    rusanov_pair<D>(qm, qp, j, G.gamma, G.gm1, dlow, dhigh);
  }
}
template <int D, int SYS>
__device__ __forceinline__ void lim_cons_to_prim(const double* q, double gm1, double* v) {
  if constexpr (SYS == 1) v[0] = q[0];
  else cons_to_prim<D>(q, gm1, v);
}
template <int D, int SYS>
__device__ __forceinline__ void lim_prim_to_cons(const double* v, double gm1, double* q) {
  if constexpr (SYS == 1) q[0] = v[0];
  else prim_to_cons<D>(v, gm1, q);
}

// map a global subcell coordinate along axis j into the grid; returns false
// for kinds without a device mapping (exact / ghost); *flip toggles for walls
__device__ __forceinline__ bool map_axis(int64_t g, int64_t nS, int bc_lo, int bc_hi,
                                         int64_t* out, bool* flip) {
  if (g >= 0 && g < nS) {
    *out = g;
    return true;
  }
  const int kind = g < 0 ? bc_lo : bc_hi;
  if (kind == ADG_BC_PERIODIC) {
    int64_t r = g % nS;
    *out = r < 0 ? r + nS : r;
    return true;
  }
  if (kind == ADG_BC_OUTFLOW) {
    *out = g < 0 ? 0 : nS - 1;
    return true;
  }
  if (kind == ADG_BC_WALL) {
    *out = g < 0 ? -1 - g : 2 * nS - 1 - g;
    *flip = !*flip;
    return true;
  }
  return false;
}

// prev_sub value set (m doubles) at global subcell coordinate gs[] of the
// padded field.  The reference pads axis 0 first, then axis 1 on the padded
// field, then axis 2 (driver.py:301-315), so the axes are resolved from the
// last padded one down: periodic / outflow / wall map the coordinate into
// the grid (wall: mirror + normal-momentum flip); an exact face reads the
// caller's slab, which was evaluated at the raw coordinates of the axes
// padded before it (corners included) and the mapped ones of those after.
template <int D, int P, int SYS>
__device__ __forceinline__ void fetch_sub(const double* __restrict__ sub, const LimGrid& G,
                                          const int64_t* gs, double* out) {
  using C = LimCfg<D, P, SYS>;
  constexpr int S = C::S, M = C::M;
  int64_t g[3] = {0, 0, 0};
  bool flip[3] = {false, false, false};
#pragma unroll
  for (int j = 0; j < D; ++j) g[j] = gs[j];
  const double* p = nullptr;
#pragma unroll
  for (int j = D - 1; j >= 0; --j) {
    const int64_t nS = G.n[j] * S;
    if (g[j] >= 0 && g[j] < nS) continue;
    const int side = g[j] >= nS ? 1 : 0;
    if (G.bc[j][side] == ADG_BC_GHOST) {
      int64_t off = 0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const int64_t ni = G.n[i] * S;
        int64_t len, idx;
        if (i < j) {
          len = ni + 2 * G.L;
          idx = g[i] + G.L;
        } else if (i == j) {
          len = G.L;
          idx = side ? g[i] - ni : g[i] + G.L;
        } else {
          len = ni;
          idx = g[i];
        }
        off = off * len + idx;
      }
      p = G.slab[j][side] + (size_t)off * M;
      break;
    }
    map_axis(g[j], nS, G.bc[j][0], G.bc[j][1], &g[j], &flip[j]);
  }
  if (!p) {
    int64_t cc[3], loc[3];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      cc[j] = g[j] / S;
      loc[j] = g[j] - cc[j] * S;
    }
    const int64_t e = cell_index<D>(cc, G.n);
    int s = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) s = s * S + (int)loc[j];
    p = sub + ((size_t)e * C::SD + s) * M;
  }
#pragma unroll
  for (int v = 0; v < M; ++v) out[v] = p[v];
  if constexpr (SYS == 0) {   // reflect (systems.py:231-234); advection: identity
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (flip[j]) out[1 + j] = -out[1 + j];
  }
}

// subcell averages of one cell's nodal data held in shared memory:
// sequential per-axis contraction with P_sub (limiter.py:27-33)
// WARP = true: the calling warp alone does the cell (tid = lane, nt = 32)
// Ps: the projection matrix P_sub [S][P] staged in shared memory (the
// lanes of a pass index different rows: constant-bank reads would replay
// once per distinct row); null -> the constant tables
template <int D, int P, int SYS, bool WARP = false, bool SPS = false>
__device__ void project_cell(const double* __restrict__ nodal, double* __restrict__ tmp,
                             double* __restrict__ out, int tid, int nt,
                             const double* __restrict__ Ps = nullptr) {
  using C = LimCfg<D, P, SYS>;
  constexpr int S = C::S, M = C::M;
  const DegreeTables& T = tab<P>();
  auto pm = [&](int idx) { return SPS ? Ps[idx] : T.sub_project[idx]; };
  if (D == 1) {
    for (int x = tid; x < S * M; x += nt) {
      const int s = x / M, v = x - s * M;
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < P; ++i) acc = fma(pm(s * P + i), nodal[i * M + v], acc);
      out[x] = acc;
    }
    return;
  }
  if (D == 2 && WARP) {
    // one warp per cell: lanes own (i1, v) columns, then (s0, v) rows, and
    // every P_sub coefficient is a compile-time constant-bank operand (same
    // fma order per output as the generic passes below)
    for (int x = tid; x < P * M; x += 32) {
      const int i1 = x / M, v = x - (x / M) * M;
      double col[P];
#pragma unroll
      for (int i0 = 0; i0 < P; ++i0) col[i0] = nodal[(i0 * P + i1) * M + v];
#pragma unroll
      for (int s0 = 0; s0 < S; ++s0) {
        double acc = 0.0;
#pragma unroll
        for (int i0 = 0; i0 < P; ++i0) acc = fma(T.sub_project[s0 * P + i0], col[i0], acc);
        tmp[(s0 * P + i1) * M + v] = acc;
      }
    }
    __syncwarp();
    for (int x = tid; x < S * M; x += 32) {
      const int s0 = x / M, v = x - (x / M) * M;
      double row[P];
#pragma unroll
      for (int i1 = 0; i1 < P; ++i1) row[i1] = tmp[(s0 * P + i1) * M + v];
#pragma unroll
      for (int s1 = 0; s1 < S; ++s1) {
        double acc = 0.0;
#pragma unroll
        for (int i1 = 0; i1 < P; ++i1) acc = fma(T.sub_project[s1 * P + i1], row[i1], acc);
        out[(s0 * S + s1) * M + v] = acc;
      }
    }
    return;
  }
  if (D == 2) {
    // axis 0: tmp[s0][i1][v]
    for (int x = tid; x < S * P * M; x += nt) {
      const int s0 = x / (P * M), r = x - s0 * P * M, i1 = r / M, v = r - i1 * M;
      double acc = 0.0;
#pragma unroll
      for (int i0 = 0; i0 < P; ++i0)
        acc = fma(pm(s0 * P + i0), nodal[(i0 * P + i1) * M + v], acc);
      tmp[x] = acc;
    }
    if (WARP) __syncwarp(); else __syncthreads();
    for (int x = tid; x < S * S * M; x += nt) {
      const int s0 = x / (S * M), r = x - s0 * S * M, s1 = r / M, v = r - s1 * M;
      double acc = 0.0;
#pragma unroll
      for (int i1 = 0; i1 < P; ++i1)
        acc = fma(pm(s1 * P + i1), tmp[(s0 * P + i1) * M + v], acc);
      out[x] = acc;
    }
    return;
  }
  // D == 3: three passes through tmp (size S*S*P*M) using out as scratch
  for (int x = tid; x < S * P * P * M; x += nt) {
    const int s0 = x / (P * P * M), r = x - s0 * P * P * M;
    double acc = 0.0;
#pragma unroll
    for (int i0 = 0; i0 < P; ++i0) acc = fma(pm(s0 * P + i0), nodal[i0 * P * P * M + r], acc);
    out[x] = acc;
  }
  if (WARP) __syncwarp(); else __syncthreads();
  for (int x = tid; x < S * S * P * M; x += nt) {
    const int s0 = x / (S * P * M), r = x - s0 * S * P * M, s1 = r / (P * M),
              r2 = r - s1 * P * M;
    double acc = 0.0;
#pragma unroll
    for (int i1 = 0; i1 < P; ++i1)
      acc = fma(pm(s1 * P + i1), out[(s0 * P + i1) * P * M + r2], acc);
    tmp[x] = acc;
  }
  if (WARP) __syncwarp(); else __syncthreads();
  for (int x = tid; x < S * S * S * M; x += nt) {
    const int s01 = x / (S * M), r = x - s01 * S * M, s2 = r / M, v = r - s2 * M;
    double acc = 0.0;
#pragma unroll
    for (int i2 = 0; i2 < P; ++i2)
      acc = fma(pm(s2 * P + i2), tmp[(s01 * P + i2) * M + v], acc);
    out[x] = acc;
  }
}

template <int D, int P, int SYS>
__device__ __forceinline__ size_t proj_scratch() {
  using C = LimCfg<D, P, SYS>;
  return D == 3 ? (size_t)C::S * C::S * P * C::M : (size_t)C::S * P * C::M;
}

// -------------------------------------------------------------- kernels
// Limiter screening is one warp per cell: a cell's projection is a few
// hundred short dot products, so a warp keeps all lanes busy without
// block-wide barriers, and 8 cells share a CTA.
template <int D, int P, int SYS>
struct WarpCfg {
  using C = LimCfg<D, P, SYS>;
  static constexpr int SCR = D == 3 ? C::S * C::S * P * C::M : C::S * P * C::M;
  static constexpr int OUT = (D == 3 ? C::S * P * P * C::M : 0) > C::SD * C::M
                                 ? C::S * P * P * C::M : C::SD * C::M;
  // (the second nodal block: the next cell's candidate lands there by
  // cp.async while the warp screens the current one, adg_detect)
  static constexpr int NOD2 = C::PD * C::M;
  static constexpr int PER_WARP = C::PD * C::M + OUT + SCR + 2 * C::M + NOD2;   // doubles
  static constexpr int W0 = (200 * 1024) / (PER_WARP * 8);
  static constexpr int WPB = W0 >= 8 ? 8 : (W0 >= 1 ? W0 : 1);   // warps (cells) per CTA
  static constexpr int PS = ((C::S * P + 1) / 2) * 2;   // staged P_sub (16-byte multiple)
  static constexpr size_t SMEM = ((size_t)WPB * PER_WARP + PS) * 8;
  // tiles beyond shared memory (3-D, N >= 3): per-block slices of an
  // L2-resident global scratch, 4 warps (cells) per block
  static constexpr bool GS = SMEM > 227 * 1024;
  static constexpr int WPBX = GS ? 4 : WPB;
  static constexpr size_t BLOCK_DBL = (size_t)WPBX * PER_WARP + PS;
  // adg_detect: compiled for three CTAs per SM where shared memory allows
  // them (80 instead of 106 registers at 2-D N = 5: C4 step 4.42 -> 4.30 ms)
  static constexpr int DET_MINB = (!GS && 3 * (SMEM + 1024) <= 228 * 1024) ? 3 : 1;
};

// P_sub of this degree into the CTA's shared copy (before any warp uses it)
template <int D, int P, int SYS>
__device__ __forceinline__ const double* stage_psub(double* dst) {
  using C = LimCfg<D, P, SYS>;
  const DegreeTables& T = tab<P>();
  for (int x = threadIdx.x; x < C::S * P; x += blockDim.x) dst[x] = T.sub_project[x];
  __syncthreads();
  return dst;
}

// per-block scratch of the block-per-cell kernels (doubles); above 227 KB
// they run on an L2-resident global scratch instead of shared memory
template <int D, int P, int SYS>
struct LimDbl {
  using C = LimCfg<D, P, SYS>;
  static constexpr size_t TMP = D == 3 ? (size_t)P * C::S * C::S * C::M + (size_t)P * P * C::S * C::M
                                       : (size_t)P * C::S * C::M;
  static constexpr size_t RESCUE = (size_t)C::WD * C::M + (size_t)C::RD * C::M * (1 + D) +
                                   (size_t)C::SD * C::M + TMP + (size_t)C::SD * C::M +
                                   (size_t)C::PD * C::M + 64;
  static constexpr size_t RECOVER = (size_t)C::SD * C::M + (size_t)C::PD * C::M + TMP;
  static constexpr size_t POUT = D == 3 ? (size_t)C::S * P * P * C::M : (size_t)C::SD * C::M;
  static constexpr size_t PTMP = D == 3 ? (size_t)C::S * C::S * P * C::M : (size_t)C::S * P * C::M;
  static constexpr size_t PROJ = (size_t)C::PD * C::M +
                                 (POUT > (size_t)C::SD * C::M ? POUT : (size_t)C::SD * C::M) + PTMP;
  static constexpr size_t LIM = 227 * 1024 / 8;
};

// per-cell subcell averages + extrema of nodal data staged in a warp's
// shared slice; writes sub / cmin / cmax of cell e when they are non-null
template <int D, int P, int SYS>
__device__ __forceinline__ void warp_project_store(double* nodal, double* out, double* tmp,
                                                   int lane, int64_t e, double* sub,
                                                   double* cmin, double* cmax,
                                                   const double* Ps) {
  using C = LimCfg<D, P, SYS>;
  constexpr int M = C::M, SD = C::SD;
  project_cell<D, P, SYS, true, true>(nodal, tmp, out, lane, 32, Ps);
  __syncwarp();
  if (sub)
    for (int x = lane; x < SD * M; x += 32) sub[(size_t)e * SD * M + x] = out[x];
  if (cmin) {
#pragma unroll
    for (int v = 0; v < M; ++v) {
      double lo = __longlong_as_double(0x7ff0000000000000LL), hi = -lo;
      for (int x = lane; x < SD; x += 32) {
        lo = fmin(lo, out[x * M + v]);
        hi = fmax(hi, out[x * M + v]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      if (lane == 0) {
        cmin[e * M + v] = lo;
        cmax[e * M + v] = hi;
      }
    }
  }
}

// prev_sub + per-cell extrema of u^n
template <int D, int P, int SYS>
__global__ void __launch_bounds__(WarpCfg<D, P, SYS>::WPBX * 32)
subcell_prep_kernel(const double* __restrict__ u, int64_t E, double* __restrict__ sub,
                    double* __restrict__ cmin, double* __restrict__ cmax, double* gscr) {
  using C = LimCfg<D, P, SYS>;
  using W = WarpCfg<D, P, SYS>;
  constexpr int M = C::M, PD = C::PD;
  extern __shared__ __align__(16) double lsm_s[];
  double* lsm = W::GS ? gscr + (size_t)blockIdx.x * W::BLOCK_DBL : lsm_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* Ps = stage_psub<D, P, SYS>(lsm + W::WPBX * W::PER_WARP);
  double* nodal = lsm + warp * W::PER_WARP;
  double* out = nodal + PD * M;
  double* tmp = out + W::OUT;
  for (int64_t e = (int64_t)blockIdx.x * W::WPBX + warp; e < E; e += (int64_t)gridDim.x * W::WPBX) {
    for (int x = lane; x < PD * M; x += 32) nodal[x] = u[(size_t)e * PD * M + x];
    __syncwarp();
    warp_project_store<D, P, SYS>(nodal, out, tmp, lane, e, sub, cmin, cmax, Ps);
    __syncwarp();
  }
}

// min/max over the ghost cell beyond face (axis j, side) of cell c: the
// reference pads S subcell layers through the face kind (driver.py:317-340)
template <int D, int P, int SYS>
__device__ void ghost_extrema(const double* __restrict__ sub, const double* __restrict__ cmin,
                              const double* __restrict__ cmax, const LimGrid& G,
                              const int64_t* c, int j, int side, double* lo, double* hi) {
  using C = LimCfg<D, P, SYS>;
  constexpr int S = C::S, M = C::M;
  const int kind = G.bc[j][side];
  int64_t cc[3] = {c[0], c[1], c[2]};
  if (kind == ADG_BC_PERIODIC) {
    cc[j] = side ? 0 : G.n[j] - 1;
    const int64_t e = cell_index<D>(cc, G.n);
#pragma unroll
    for (int v = 0; v < M; ++v) {
      lo[v] = cmin[e * M + v];
      hi[v] = cmax[e * M + v];
    }
    return;
  }
  if (kind == ADG_BC_GHOST) {
    // exact: the S^d caller-evaluated subcells of the ghost cell
#pragma unroll
    for (int v = 0; v < M; ++v) {
      lo[v] = __longlong_as_double(0x7ff0000000000000LL);
      hi[v] = -lo[v];
    }
    for (int s = 0; s < C::SD; ++s) {
      int rem = s;
      int64_t gs[3] = {0, 0, 0};
      for (int a = D - 1; a >= 0; --a) {
        const int ia = rem % S;
        rem /= S;
        gs[a] = a == j ? (side ? G.n[j] * S + ia : ia - S) : c[a] * S + ia;
      }
      double q[M];
      fetch_sub<D, P, SYS>(sub, G, gs, q);
#pragma unroll
      for (int v = 0; v < M; ++v) {
        lo[v] = fmin(lo[v], q[v]);
        hi[v] = fmax(hi[v], q[v]);
      }
    }
    return;
  }
  const int64_t e = cell_index<D>(cc, G.n);   // the edge cell itself
  if (kind == ADG_BC_WALL) {
#pragma unroll
    for (int v = 0; v < M; ++v) {
      lo[v] = cmin[e * M + v];
      hi[v] = cmax[e * M + v];
    }
    if constexpr (SYS == 0) {
      const double a = lo[1 + j], b = hi[1 + j];
      lo[1 + j] = -b;
      hi[1 + j] = -a;
    }
    return;
  }
  // outflow: every ghost layer repeats the edge subcell layer
#pragma unroll
  for (int v = 0; v < M; ++v) {
    lo[v] = __longlong_as_double(0x7ff0000000000000LL);
    hi[v] = -lo[v];
  }
  const int edge = side ? S - 1 : 0;
  for (int s = 0; s < C::SD; ++s) {
    int rem = s, idx[3] = {0, 0, 0};
    for (int a = D - 1; a >= 0; --a) {
      idx[a] = rem % S;
      rem /= S;
    }
    if (idx[j] != edge) continue;
    const double* p = sub + ((size_t)e * C::SD + s) * M;
#pragma unroll
    for (int v = 0; v < M; ++v) {
      lo[v] = fmin(lo[v], p[v]);
      hi[v] = fmax(hi[v], p[v]);
    }
  }
}

// troubled-cell screen (limiter.py:51-86, driver.py:272-285), one warp per
// cell.  The candidate's subcell averages and extrema are written to
// sub_out / cmin_out / cmax_out (when non-null): for every cell the rescue
// leaves alone they are exactly the next step's prev_sub, so the driver
// skips the separate projection of u^(n+1).
template <int D, int P, int SYS>
__global__ void __launch_bounds__(WarpCfg<D, P, SYS>::WPBX * 32, WarpCfg<D, P, SYS>::DET_MINB)
detect_kernel(const double* __restrict__ prev_sub, const double* __restrict__ cmin,
              const double* __restrict__ cmax, const double* __restrict__ cand,
              const uint8_t* __restrict__ pred_bad, LimGrid G, int64_t E, double delta0,
              double eps, int force_all, uint8_t* __restrict__ troubled, int32_t* idx,
              int32_t* count, double* __restrict__ sub_out, double* __restrict__ cmin_out,
              double* __restrict__ cmax_out, double* gscr) {
  using C = LimCfg<D, P, SYS>;
  using W = WarpCfg<D, P, SYS>;
  constexpr int M = C::M, SD = C::SD, PD = C::PD;
  extern __shared__ __align__(16) double lsm_s[];
  double* lsm = W::GS ? gscr + (size_t)blockIdx.x * W::BLOCK_DBL : lsm_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* Ps = stage_psub<D, P, SYS>(lsm + W::WPBX * W::PER_WARP);
  double* nod0 = lsm + warp * W::PER_WARP;
  double* out = nod0 + PD * M;
  double* tmp = out + W::OUT;
  double* s_lo = tmp + W::SCR;
  double* s_hi = s_lo + M;
  double* nod1 = s_hi + M;
  // the candidate of the warp's NEXT cell is fetched (cp.async) while the
  // current one is screened: the synchronous load held 29 % of the kernel's
  // stall samples at C4 (global-scratch variant: plain loads)
  constexpr bool PF = !W::GS;
  const int64_t estride = (int64_t)gridDim.x * W::WPBX;
  auto prefetch = [&](int64_t ee, double* dst) {
    const double* src = cand + (size_t)ee * PD * M;
    for (int x = lane; x < PD * M; x += 32) cp_async8(dst + x, src + x);
    cp_async_commit();
  };
  int64_t e0 = (int64_t)blockIdx.x * W::WPBX + warp;
  if (PF && e0 < E) prefetch(e0, nod0);
  int par = 0;
  for (int64_t e = e0; e < E; e += estride, par ^= 1) {
    double* nodal = PF && par ? nod1 : nod0;
    if (PF) {
      if (e + estride < E) {
        prefetch(e + estride, par ? nod0 : nod1);
        cp_async_wait_1();
      } else {
        cp_async_wait_all();
      }
      __syncwarp();
    } else {
      for (int x = lane; x < PD * M; x += 32) nodal[x] = cand[(size_t)e * PD * M + x];
    }
    // DMP bounds: lane v < M owns quantity v; own cell, then the face
    // neighbours in axis order, low then high (min / max are order-free)
    int64_t c[3] = {0, 0, 0};
    {
      int64_t r = e;
#pragma unroll
      for (int j = D - 1; j >= 0; --j) {
        c[j] = r % G.n[j];
        r /= G.n[j];
      }
    }
    const int vq = lane < M ? lane : 0;
    double lo = cmin[e * M + vq], hi = cmax[e * M + vq];
    // interior face neighbours: every load issued before any is folded
    double nlo[2 * D], nhi[2 * D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const bool inside = side ? (c[j] + 1 < G.n[j]) : (c[j] > 0);
        int64_t en = e;
        if (inside) {
          en = 0;
#pragma unroll
          for (int a = 0; a < D; ++a) en = en * G.n[a] + c[a] + (a == j ? (side ? 1 : -1) : 0);
        }
        nlo[2 * j + side] = cmin[en * M + vq];
        nhi[2 * j + side] = cmax[en * M + vq];
      }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const bool inside = side ? (c[j] + 1 < G.n[j]) : (c[j] > 0);
        if (inside) {
          lo = fmin(lo, nlo[2 * j + side]);
          hi = fmax(hi, nhi[2 * j + side]);
        } else {   // warp-uniform: a boundary face of this cell
          if (lane == 0) ghost_extrema<D, P, SYS>(prev_sub, cmin, cmax, G, c, j, side, s_lo, s_hi);
          __syncwarp();
          lo = fmin(lo, s_lo[vq]);
          hi = fmax(hi, s_hi[vq]);
          __syncwarp();
        }
      }
    }
    {
      const double delta = fmax(delta0, eps * (hi - lo));
      if (lane < M) {
        s_lo[lane] = lo - delta;
        s_hi[lane] = hi + delta;
      }
    }
    __syncwarp();
    warp_project_store<D, P, SYS>(nodal, out, tmp, lane, e, sub_out, cmin_out, cmax_out, Ps);
    int bad = lane == 0 ? (force_all || pred_bad[e]) : 0;
    for (int x = lane; x < SD; x += 32) {
      const double* q = out + x * M;
#pragma unroll
      for (int v = 0; v < M; ++v) bad |= (q[v] < s_lo[v]) | (q[v] > s_hi[v]);
      bad |= !lim_adm_fast<D, SYS>(q, G.gm1);
    }
    for (int nd = lane; nd < PD; nd += 32) bad |= !lim_adm_fast<D, SYS>(nodal + nd * M, G.gm1);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      troubled[e] = (uint8_t)bad;
      if (bad) idx[atomicAdd(count, 1)] = (int32_t)e;
    }
    __syncwarp();
  }
}

// Rusanov one-sided terms (corrector.py:100-129) live in adg_common.cuh
// face states of the primitive-mode half step back to conservative
// (limiter.py:160-171)
template <int D, int SYS>
__device__ __forceinline__ void to_cons2(double* a, double* b, double gm1) {
  if constexpr (SYS == 0) {
    constexpr int M = D + 2;
    double t[M];
    prim_to_cons<D>(a, gm1, t);
#pragma unroll
    for (int v = 0; v < M; ++v) a[v] = t[v];
    prim_to_cons<D>(b, gm1, t);
#pragma unroll
    for (int v = 0; v < M; ++v) b[v] = t[v];
  }
}

// nodal polynomial of one cell from its S^d subcell averages
// (recover_from_subcells, limiter.py:36-42): sequential per-axis
// contraction with R_sub; tmp needs P S^(D-1) m (+ P^2 S m for D = 3) doubles
template <int D, int P, int SYS>
__device__ void recover_cell(const double* __restrict__ nw, double* __restrict__ tmp,
                             double* __restrict__ nod, int tid, int NT) {
  using C = LimCfg<D, P, SYS>;
  constexpr int M = C::M, S = C::S, PD = C::PD;
  const DegreeTables& T = tab<P>();
    if (D == 1) {
      for (int x = tid; x < PD * M; x += NT) {
        const int i = x / M, v = x - i * M;
        double acc = 0.0;
        for (int s = 0; s < S; ++s) acc = fma(T.sub_recover[i * S + s], nw[s * M + v], acc);
        nod[x] = acc;
      }
    } else if (D == 2) {
      for (int x = tid; x < P * S * M; x += NT) {
        const int i0 = x / (S * M), r = x - i0 * S * M;
        double acc = 0.0;
        for (int s0 = 0; s0 < S; ++s0) acc = fma(T.sub_recover[i0 * S + s0], nw[s0 * S * M + r], acc);
        tmp[x] = acc;
      }
      __syncthreads();
      for (int x = tid; x < PD * M; x += NT) {
        const int i0 = x / (P * M), r = x - i0 * P * M, i1 = r / M, v = r - i1 * M;
        double acc = 0.0;
        for (int s1 = 0; s1 < S; ++s1)
          acc = fma(T.sub_recover[i1 * S + s1], tmp[(i0 * S + s1) * M + v], acc);
        nod[x] = acc;
      }
    } else {
      for (int x = tid; x < P * S * S * M; x += NT) {
        const int i0 = x / (S * S * M), r = x - i0 * S * S * M;
        double acc = 0.0;
        for (int s0 = 0; s0 < S; ++s0)
          acc = fma(T.sub_recover[i0 * S + s0], nw[s0 * S * S * M + r], acc);
        tmp[x] = acc;
      }
      __syncthreads();
      double* t2 = tmp + P * S * S * M;
      for (int x = tid; x < P * P * S * M; x += NT) {
        const int i0 = x / (P * S * M), r = x - i0 * P * S * M, i1 = r / (S * M),
                  r2 = r - i1 * S * M;
        double acc = 0.0;
        for (int s1 = 0; s1 < S; ++s1)
          acc = fma(T.sub_recover[i1 * S + s1], tmp[(i0 * S + s1) * S * M + r2], acc);
        t2[x] = acc;
      }
      __syncthreads();
      for (int x = tid; x < PD * M; x += NT) {
        const int i01 = x / (P * M), r = x - i01 * P * M, i2 = r / M, v = r - i2 * M;
        double acc = 0.0;
        for (int s2 = 0; s2 < S; ++s2)
          acc = fma(T.sub_recover[i2 * S + s2], t2[(i01 * S + s2) * M + v], acc);
        nod[x] = acc;
      }
    }
}

// MUSCL-Hancock rescue of one troubled cell per block (limiter.py:104-223).
// WIN = 0: the cell's window is gathered from the t^n subcell field (the
// driver path); recovery + flattening write u_out and a failure raises
// *failed.  WIN = 1: muscl_subcell_step on caller windows (limiter.py:104-121):
// window b is windows[b], the new averages go to avg_out[b] and the
// per-window failure flag to fail_each[b].
template <int D, int P, int SYS, int WIN>
__global__ void __launch_bounds__(LimCfg<D, P, SYS>::NT)
rescue_kernel(const double* __restrict__ prev_sub, const int32_t* __restrict__ idx,
              const int32_t* __restrict__ count, LimGrid G, const double* __restrict__ dt_dev,
              double* __restrict__ u_out, int32_t* failed, const double* __restrict__ windows,
              double* __restrict__ avg_out, uint8_t* __restrict__ fail_each,
              double* __restrict__ sub_next, double* __restrict__ cmin_next,
              double* __restrict__ cmax_next, double* gscr) {
  using C = LimCfg<D, P, SYS>;
  constexpr int M = C::M, S = C::S, SD = C::SD, PD = C::PD, W = C::W, WD = C::WD, R = C::R,
                RD = C::RD, NT = C::NT;
  const DegreeTables& T = tab<P>();
  constexpr bool GS = LimDbl<D, P, SYS>::RESCUE > LimDbl<D, P, SYS>::LIM;
  extern __shared__ __align__(16) double lsm_s[];
  double* lsm = GS ? gscr + (size_t)blockIdx.x * LimDbl<D, P, SYS>::RESCUE : lsm_s;
  double* win = lsm;                    // [WD][M]
  double* vh = win + WD * M;            // [RD][M]  half-step states
  double* sl = vh + RD * M;             // [RD][D][M] limited slopes
  double* nw = sl + RD * D * M;         // [SD][M]  new averages
  double* tmp = nw + SD * M;            // recovery scratch
  double* nod = tmp + (D == 3 ? S * S * P * M : S * P * M) + SD * M;  // [PD][M]
  __shared__ int s_ok, s_flat;
  const int tid = threadIdx.x;
  const double dt = *dt_dev;
  const int ncells = *count;
  for (int b = blockIdx.x; b < ncells; b += gridDim.x) {
    const int64_t e = WIN ? b : idx[b];
    int64_t c[3] = {0, 0, 0};
    if (!WIN) {
      int64_t r = e;
      for (int j = D - 1; j >= 0; --j) {
        c[j] = r % G.n[j];
        r /= G.n[j];
      }
    }
    // window of t^n subcell averages with a 2-layer halo (limiter.py:89-101)
    for (int w = tid; w < WD; w += NT) {
      if (WIN) {
#pragma unroll
        for (int v = 0; v < M; ++v) win[w * M + v] = windows[((size_t)b * WD + w) * M + v];
      } else {
        int rem = w;
        int64_t gs[3] = {0, 0, 0};
        for (int j = D - 1; j >= 0; --j) {
          gs[j] = c[j] * S - 2 + rem % W;
          rem /= W;
        }
        fetch_sub<D, P, SYS>(prev_sub, G, gs, win + w * M);
      }
      if (G.prim) {   // limiter.py:127-128: the window in primitive variables
        double vv[M];
        lim_cons_to_prim<D, SYS>(win + w * M, G.gm1, vv);
#pragma unroll
        for (int v = 0; v < M; ++v) win[w * M + v] = vv[v];
      }
    }
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {   // sloped, then first order
      const bool flat = pass == 1;
      if (tid == 0) s_ok = 1;
      __syncthreads();
      // slopes + half step on the 1-halo region
      for (int r = tid; r < RD; r += NT) {
        int ri[3] = {0, 0, 0}, rem = r;
        for (int j = D - 1; j >= 0; --j) {
          ri[j] = rem % R;
          rem /= R;
        }
        auto wix = [&](int dj, int off) {
          int x = 0;
          for (int j = 0; j < D; ++j) x = x * W + ri[j] + 1 + (j == dj ? off : 0);
          return x;
        };
        const double* cq = win + wix(0, 0) * M;
        double slope[D][M];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double* up = win + wix(j, 1) * M;
          const double* dn = win + wix(j, -1) * M;
#pragma unroll
          for (int v = 0; v < M; ++v) {
            if (flat) {
              slope[j][v] = 0.0;
            } else {
              const double fwd = (up[v] - cq[v]) / G.h[j];
              const double bwd = (cq[v] - dn[v]) / G.h[j];
              slope[j][v] = minmod(fwd, bwd);
            }
          }
        }
        double rate[M];
#pragma unroll
        for (int v = 0; v < M; ++v) rate[v] = 0.0;
        if (G.prim) {
          // limiter.py:146-147: half = c + dt/2 primitive_rhs(c, slopes)
          if constexpr (SYS == 0) primitive_rhs<D>(cq, slope, G.gamma, rate);
        } else {
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double qh[M], ql[M], fh[M], fl[M];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            const double off = 0.5 * G.h[j] * slope[j][v];
            qh[v] = cq[v] + off;
            ql[v] = cq[v] - off;
          }
          lim_flux<D, SYS>(qh, G, j, fh);
          lim_flux<D, SYS>(ql, G, j, fl);
#pragma unroll
          for (int v = 0; v < M; ++v) rate[v] = rate[v] - (fh[v] - fl[v]) / G.h[j];
        }
        }
        double half[M];
#pragma unroll
        for (int v = 0; v < M; ++v) {
          half[v] = cq[v] + (0.5 * dt) * rate[v];
          vh[r * M + v] = half[v];
        }
        bool ok = true;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double lo[M], hi[M];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            const double off = 0.5 * G.h[j] * slope[j][v];
            sl[(r * D + j) * M + v] = off;
            lo[v] = half[v] - off;
            hi[v] = half[v] + off;
          }
          if (G.prim) {
            double tq[M];
            lim_prim_to_cons<D, SYS>(lo, G.gm1, tq);
#pragma unroll
            for (int v = 0; v < M; ++v) lo[v] = tq[v];
            lim_prim_to_cons<D, SYS>(hi, G.gm1, tq);
#pragma unroll
            for (int v = 0; v < M; ++v) hi[v] = tq[v];
          }
          ok = ok && lim_adm<D, SYS>(lo, G.gm1) && lim_adm<D, SYS>(hi, G.gm1);
        }
        if (!ok) s_ok = 0;
      }
      __syncthreads();
      // core update through the subcell faces
      for (int s = tid; s < SD; s += NT) {
        int si[3] = {0, 0, 0}, rem = s;
        for (int j = D - 1; j >= 0; --j) {
          si[j] = rem % S;
          rem /= S;
        }
        auto rix = [&](int dj, int off) {
          int x = 0;
          for (int j = 0; j < D; ++j) x = x * R + si[j] + 1 + (j == dj ? off : 0);
          return x;
        };
        auto wcore = [&]() {
          int x = 0;
          for (int j = 0; j < D; ++j) x = x * W + si[j] + 2;
          return x;
        };
        double q[M];
        if (G.prim && WIN) {   // conservative core average (limiter.py:178)
#pragma unroll
          for (int v = 0; v < M; ++v) q[v] = windows[((size_t)b * WD + wcore()) * M + v];
        } else if (G.prim) {
          int64_t gs[3] = {0, 0, 0};
          for (int j = 0; j < D; ++j) gs[j] = c[j] * S + si[j];
          fetch_sub<D, P, SYS>(prev_sub, G, gs, q);
        } else {
#pragma unroll
          for (int v = 0; v < M; ++v) q[v] = win[wcore() * M + v];
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const int rc = rix(0, 0), rl = rix(j, -1), rh = rix(j, 1);
          double a[M], bq[M], dlo_h[M], dhi_h[M], dlo_l[M], dhi_l[M];
          // high face: minus = hi state of this cell, plus = lo state of next
#pragma unroll
          for (int v = 0; v < M; ++v) {
            a[v] = vh[rc * M + v] + sl[(rc * D + j) * M + v];
            bq[v] = vh[rh * M + v] - sl[(rh * D + j) * M + v];
          }
          if (G.prim) to_cons2<D, SYS>(a, bq, G.gm1);
          lim_rusanov<D, SYS>(a, bq, j, G, dlo_h, dhi_h);
          // low face: minus = hi state of previous, plus = lo state of this
#pragma unroll
          for (int v = 0; v < M; ++v) {
            a[v] = vh[rl * M + v] + sl[(rl * D + j) * M + v];
            bq[v] = vh[rc * M + v] - sl[(rc * D + j) * M + v];
          }
          if (G.prim) to_cons2<D, SYS>(a, bq, G.gm1);
          lim_rusanov<D, SYS>(a, bq, j, G, dlo_l, dhi_l);
          const double c_j = dt / G.h[j];
#pragma unroll
          for (int v = 0; v < M; ++v) q[v] -= c_j * (dlo_h[v] + dhi_l[v]);
        }
        if (!lim_adm<D, SYS>(q, G.gm1)) s_ok = 0;
#pragma unroll
        for (int v = 0; v < M; ++v) nw[s * M + v] = q[v];
      }
      __syncthreads();
      if (s_ok) break;
      if (pass == 1 && !WIN) {
        if (tid == 0) atomicOr(failed, 1);
      }
      __syncthreads();
    }
    if (WIN) {
      for (int x = tid; x < SD * M; x += NT) avg_out[(size_t)b * SD * M + x] = nw[x];
      if (tid == 0) fail_each[b] = !s_ok;
      __syncthreads();
      continue;
    }
    if (!s_ok) {
      __syncthreads();
      continue;
    }
    recover_cell<D, P, SYS>(nw, tmp, nod, tid, NT);
    __syncthreads();
    // flatten_inadmissible (limiter.py:205-223): nodal and its subcell
    // projection must be admissible, else the cell becomes its mean
    if (tid == 0) s_flat = 0;
    __syncthreads();
    for (int nd = tid; nd < PD; nd += NT)
      if (!lim_adm<D, SYS>(nod + nd * M, G.gm1)) s_flat = 1;
    __syncthreads();
    if (!s_flat) {
      double* pj = vh;    // reuse: projection of the recovered polynomial
      project_cell<D, P, SYS>(nod, tmp + PD * M * 0 + (D == 3 ? P * S * S * M : P * S * M), pj, tid, NT);
      __syncthreads();
      for (int s = tid; s < SD; s += NT)
        if (!lim_adm<D, SYS>(pj + s * M, G.gm1)) s_flat = 1;
      __syncthreads();
    }
    double* dst = u_out + (size_t)e * PD * M;
    if (s_flat) {
      // mean of the new subcell averages (numpy mean: sum / count)
      __shared__ double s_mean[M];
      if (tid < M) {
        double acc = 0.0;
        for (int s = 0; s < SD; ++s) acc += nw[s * M + tid];
        s_mean[tid] = acc / SD;
      }
      __syncthreads();
      for (int x = tid; x < PD * M; x += NT) nod[x] = s_mean[x % M];
    }
    for (int x = tid; x < PD * M; x += NT) dst[x] = nod[x];
    if (!WIN && sub_next) {
      // the rescued cell's subcell averages / extrema for the next step
      // (same arithmetic as the screen's projection of unrescued cells)
      __syncthreads();
      double* pj = vh;
      project_cell<D, P, SYS>(nod, tmp + (D == 3 ? P * S * S * M : P * S * M), pj, tid, NT);
      __syncthreads();
      for (int x = tid; x < SD * M; x += NT) sub_next[(size_t)e * SD * M + x] = pj[x];
      if (tid < 32) {
#pragma unroll
        for (int v = 0; v < M; ++v) {
          double lo = __longlong_as_double(0x7ff0000000000000LL), hi = -lo;
          for (int x = tid; x < SD; x += 32) {
            lo = fmin(lo, pj[x * M + v]);
            hi = fmax(hi, pj[x * M + v]);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
          }
          if (tid == 0) {
            cmin_next[e * M + v] = lo;
            cmax_next[e * M + v] = hi;
          }
        }
      }
    }
    __syncthreads();
  }
}

// recover_from_subcells (limiter.py:36-42) on E cells: ubar [E][S^d][m] ->
// nodal [E][P^d][m]
template <int D, int P, int SYS>
__global__ void __launch_bounds__(LimCfg<D, P, SYS>::NT)
recover_kernel(const double* __restrict__ ubar, int64_t E, double* __restrict__ out,
               double* gscr) {
  using C = LimCfg<D, P, SYS>;
  constexpr int M = C::M, SD = C::SD, PD = C::PD, NT = C::NT;
  constexpr bool GS = LimDbl<D, P, SYS>::RECOVER > LimDbl<D, P, SYS>::LIM;
  extern __shared__ __align__(16) double lsm_s[];
  double* lsm = GS ? gscr + (size_t)blockIdx.x * LimDbl<D, P, SYS>::RECOVER : lsm_s;
  double* nw = lsm;
  double* nod = nw + SD * M;
  double* tmp = nod + PD * M;
  const int tid = threadIdx.x;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    for (int x = tid; x < SD * M; x += NT) nw[x] = ubar[(size_t)e * SD * M + x];
    __syncthreads();
    recover_cell<D, P, SYS>(nw, tmp, nod, tid, NT);
    __syncthreads();
    for (int x = tid; x < PD * M; x += NT) out[(size_t)e * PD * M + x] = nod[x];
    __syncthreads();
  }
}

// flatten_inadmissible (limiter.py:205-223) on E cells, in place on nodal:
// a cell whose nodal states or their subcell projection are inadmissible
// becomes the mean of its subcell averages; *nflat counts them
template <int D, int P, int SYS>
__global__ void __launch_bounds__(LimCfg<D, P, SYS>::NT)
flatten_cells_kernel(double* __restrict__ nodal, const double* __restrict__ averages, int64_t E,
                     double gm1, int32_t* nflat, double* gscr) {
  using C = LimCfg<D, P, SYS>;
  constexpr int M = C::M, SD = C::SD, PD = C::PD, NT = C::NT;
  constexpr bool GS = LimDbl<D, P, SYS>::PROJ > LimDbl<D, P, SYS>::LIM;
  extern __shared__ __align__(16) double lsm_s[];
  double* lsm = GS ? gscr + (size_t)blockIdx.x * LimDbl<D, P, SYS>::PROJ : lsm_s;
  double* nod = lsm;
  double* pj = nod + PD * M;
  double* tmp = pj + SD * M;
  __shared__ int s_flat;
  __shared__ double s_mean[M];
  const int tid = threadIdx.x;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    double* ne = nodal + (size_t)e * PD * M;
    for (int x = tid; x < PD * M; x += NT) nod[x] = ne[x];
    if (tid == 0) s_flat = 0;
    __syncthreads();
    project_cell<D, P, SYS>(nod, tmp, pj, tid, NT);
    __syncthreads();
    int bad = 0;
    for (int nd = tid; nd < PD; nd += NT) bad |= !lim_adm<D, SYS>(nod + nd * M, gm1);
    for (int x = tid; x < SD; x += NT) bad |= !lim_adm<D, SYS>(pj + x * M, gm1);
    if (bad) s_flat = 1;
    __syncthreads();
    if (s_flat) {
      if (tid < M) {
        double acc = 0.0;
        for (int x = 0; x < SD; ++x) acc += averages[((size_t)e * SD + x) * M + tid];
        s_mean[tid] = acc / SD;
      }
      __syncthreads();
      for (int x = tid; x < PD * M; x += NT) ne[x] = s_mean[x % M];
      if (tid == 0) atomicAdd(nflat, 1);
    }
    __syncthreads();
  }
}

// IC flattening (driver.py:137-152): one block per cell
template <int D, int P, int SYS>
__global__ void __launch_bounds__(LimCfg<D, P, SYS>::NT)
flatten_ic_kernel(double* __restrict__ u, int64_t E, double gm1, int32_t* nflat,
                  double* gscr) {
  using C = LimCfg<D, P, SYS>;
  constexpr int M = C::M, SD = C::SD, PD = C::PD, NT = C::NT;
  const DegreeTables& T = tab<P>();
  constexpr bool GS = LimDbl<D, P, SYS>::PROJ > LimDbl<D, P, SYS>::LIM;
  extern __shared__ __align__(16) double lsm_s[];
  double* lsm = GS ? gscr + (size_t)blockIdx.x * LimDbl<D, P, SYS>::PROJ : lsm_s;
  double* nodal = lsm;
  double* out = nodal + PD * M;
  double* tmp = out + SD * M;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    double* ue = u + (size_t)e * PD * M;
    for (int x = tid; x < PD * M; x += NT) nodal[x] = ue[x];
    if (tid == 0) s_bad = 0;
    __syncthreads();
    project_cell<D, P, SYS>(nodal, tmp, out, tid, NT);
    __syncthreads();
    int bad = 0;
    for (int s = tid; s < SD; s += NT) bad |= !lim_adm<D, SYS>(out + s * M, gm1);
    for (int nd = tid; nd < PD; nd += NT) bad |= !lim_adm<D, SYS>(nodal + nd * M, gm1);
    if (bad) s_bad = 1;
    __syncthreads();
    if (s_bad) {
      __shared__ double s_mean[M];
      if (tid < M) {
        double acc = 0.0;
        for (int nd = 0; nd < PD; ++nd) {
          double w;
          if (D == 1) w = T.weights[nd];
          else if (D == 2) w = T.weights[nd / P] * T.weights[nd % P];
          else w = T.weights[nd / (P * P)] * T.weights[(nd / P) % P] * T.weights[nd % P];
          acc += nodal[nd * M + tid] * w;
        }
        s_mean[tid] = acc;
      }
      __syncthreads();
      for (int x = tid; x < PD * M; x += NT) ue[x] = s_mean[x % M];
      if (tid == 0) atomicAdd(nflat, 1);
    }
    __syncthreads();
  }
}

// global scratch for the kernels above (one buffer per device, grown on demand)
static double* lim_scratch(size_t bytes, std::string* err) {
  static double* ptr[64] = {};
  static size_t cap[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cap[dev] < bytes) {
    if (ptr[dev]) cudaFree(ptr[dev]);
    ptr[dev] = nullptr;
    cap[dev] = 0;
    if (cudaMalloc(&ptr[dev], bytes) != cudaSuccess) {
      *err = "limiter scratch allocation failed";
      return nullptr;
    }
    cap[dev] = bytes;
  }
  return ptr[dev];
}
constexpr int kScratchBlocks = 148 * 2;   // blocks of the global-scratch kernels

// ------------------------------------------------------------- launchers
static LimGrid lim_grid(const adg_grid* g, const adg_subcell_ghosts* gh = nullptr) {
  LimGrid G;
  for (int j = 0; j < 3; ++j)
    for (int s = 0; s < 2; ++s) G.slab[j][s] = gh ? gh->slab[j][s] : nullptr;
  G.L = gh ? gh->layers : 0;
  const int S = 2 * g->degree + 1;
  for (int j = 0; j < 3; ++j) {
    G.n[j] = j < g->dim ? g->cells[j] : 1;
    G.h[j] = j < g->dim ? g->dx[j] / S : 1.0;
    G.bc[j][0] = j < g->dim ? g->bc[j][0] : 0;
    G.bc[j][1] = j < g->dim ? g->bc[j][1] : 0;
  }
  G.gamma = g->gamma;
  G.gm1 = g->gamma - 1.0;
  G.prim = (g->system == ADG_SYS_EULER && g->mode == ADG_MODE_PRIMITIVE) ? 1 : 0;
  for (int j = 0; j < 3; ++j) G.a[j] = j < g->dim ? g->velocity[j] : 0.0;
  return G;
}

template <int D, int P, int SYS>
static size_t proj_smem() {
  using C = LimCfg<D, P, SYS>;
  const size_t out = D == 3 ? (size_t)C::S * P * P * C::M : (size_t)C::SD * C::M;
  const size_t tmp = D == 3 ? (size_t)C::S * C::S * P * C::M : (size_t)C::S * P * C::M;
  return ((size_t)C::PD * C::M + (out > (size_t)C::SD * C::M ? out : (size_t)C::SD * C::M) +
          tmp) * 8;
}

template <int D, int P, int SYS>
static size_t rescue_smem() {
  using C = LimCfg<D, P, SYS>;
  const size_t tmp = D == 3 ? (size_t)P * C::S * C::S * C::M + (size_t)P * P * C::S * C::M
                            : (size_t)P * C::S * C::M;
  return ((size_t)C::WD * C::M + (size_t)C::RD * C::M * (1 + D) + (size_t)C::SD * C::M + tmp +
          (size_t)C::SD * C::M + (size_t)C::PD * C::M + 64) * 8;
}

template <typename K>
static bool set_smem(K kern, size_t bytes) {
  if (bytes > 227 * 1024) return false;
  if (bytes > 48 * 1024)
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) ==
           cudaSuccess;
  return true;
}

static bool lim_supported(const adg_grid* g, const adg_subcell_ghosts* gh, std::string* err) {
  const int need = 2 * g->degree + 1 > 2 ? 2 * g->degree + 1 : 2;
  for (int j = 0; j < g->dim; ++j)
    for (int s = 0; s < 2; ++s)
      if (g->bc[j][s] == ADG_BC_GHOST && (!gh || !gh->slab[j][s] || gh->layers < need)) {
        *err = "ghost (exact) face without an exterior subcell slab of >= max(S, 2) layers";
        return false;
      }
  return true;
}

#define ADG_LIM_SWITCH_S(SYS_, FN, ...)                                                 \
  do {                                                                          \
    switch (g->dim * 16 + g->degree + 1) {                                      \
      case 17: rc = FN<1, 1, SYS_>(__VA_ARGS__); break;                               \
      case 18: rc = FN<1, 2, SYS_>(__VA_ARGS__); break;                               \
      case 19: rc = FN<1, 3, SYS_>(__VA_ARGS__); break;                               \
      case 20: rc = FN<1, 4, SYS_>(__VA_ARGS__); break;                               \
      case 21: rc = FN<1, 5, SYS_>(__VA_ARGS__); break;                               \
      case 22: rc = FN<1, 6, SYS_>(__VA_ARGS__); break;                               \
      case 23: rc = FN<1, 7, SYS_>(__VA_ARGS__); break;                               \
      case 24: rc = FN<1, 8, SYS_>(__VA_ARGS__); break;                               \
      case 25: rc = FN<1, 9, SYS_>(__VA_ARGS__); break;                               \
      case 26: rc = FN<1, 10, SYS_>(__VA_ARGS__); break;                              \
      case 33: rc = FN<2, 1, SYS_>(__VA_ARGS__); break;                               \
      case 34: rc = FN<2, 2, SYS_>(__VA_ARGS__); break;                               \
      case 35: rc = FN<2, 3, SYS_>(__VA_ARGS__); break;                               \
      case 36: rc = FN<2, 4, SYS_>(__VA_ARGS__); break;                               \
      case 37: rc = FN<2, 5, SYS_>(__VA_ARGS__); break;                               \
      case 38: rc = FN<2, 6, SYS_>(__VA_ARGS__); break;                               \
      case 39: rc = FN<2, 7, SYS_>(__VA_ARGS__); break;                               \
      case 40: rc = FN<2, 8, SYS_>(__VA_ARGS__); break;                               \
      case 41: rc = FN<2, 9, SYS_>(__VA_ARGS__); break;                               \
      case 42: rc = FN<2, 10, SYS_>(__VA_ARGS__); break;                              \
      case 49: rc = FN<3, 1, SYS_>(__VA_ARGS__); break;                               \
      case 50: rc = FN<3, 2, SYS_>(__VA_ARGS__); break;                               \
      case 51: rc = FN<3, 3, SYS_>(__VA_ARGS__); break;                               \
      case 52: rc = FN<3, 4, SYS_>(__VA_ARGS__); break;                               \
      case 53: rc = FN<3, 5, SYS_>(__VA_ARGS__); break;                               \
      case 54: rc = FN<3, 6, SYS_>(__VA_ARGS__); break;                               \
      case 55: rc = FN<3, 7, SYS_>(__VA_ARGS__); break;                               \
      case 56: rc = FN<3, 8, SYS_>(__VA_ARGS__); break;                               \
      case 57: rc = FN<3, 9, SYS_>(__VA_ARGS__); break;                               \
      case 58: rc = FN<3, 10, SYS_>(__VA_ARGS__); break;                              \
      default:                                                                  \
        *err = "subcell limiter on the device: unsupported dim / degree";      \
        return ADG_ERR_UNSUPPORTED;                                             \
    }                                                                           \
  } while (0)

// Euler or advection instantiation of a launcher, by the grid's plugin
#define ADG_LIM_SWITCH(FN, ...)                                                 \
  do {                                                                          \
    if (g->system == ADG_SYS_ADVECTION) ADG_LIM_SWITCH_S(1, FN, __VA_ARGS__);   \
    else ADG_LIM_SWITCH_S(0, FN, __VA_ARGS__);                                  \
  } while (0)

static int lerr(std::string* err) {
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

template <int D, int P, int SYS>
static int launch_prep(const adg_grid* g, const double* u, double* sub, double* cmin,
                       double* cmax, cudaStream_t st, std::string* err) {
  using W = WarpCfg<D, P, SYS>;
  if (!W::GS && !set_smem(subcell_prep_kernel<D, P, SYS>, W::SMEM)) {
    *err = "limiter tile exceeds shared memory";
    return ADG_ERR_UNSUPPORTED;
  }
  const int64_t E = n_elements(g);
  const int64_t nb = (E + W::WPBX - 1) / W::WPBX;
  const int64_t cap = W::GS ? kScratchBlocks : 148 * 64;
  const unsigned grid = (unsigned)(nb < cap ? nb : cap);
  double* gs = nullptr;
  if (W::GS && !(gs = lim_scratch((size_t)grid * W::BLOCK_DBL * 8, err))) return ADG_ERR_CUDA;
  subcell_prep_kernel<D, P, SYS><<<grid, W::WPBX * 32, W::GS ? 0 : W::SMEM, st>>>(u, E, sub, cmin,
                                                                           cmax, gs);
  return lerr(err);
}

template <int D, int P, int SYS>
static int launch_detect(const adg_grid* g, const double* prev_sub, const double* cmin,
                         const double* cmax, const double* cand, const uint8_t* pred_bad,
                         double d0, double eps, int force, const adg_subcell_ghosts* gh,
                         uint8_t* troubled, int32_t* idx, int32_t* count, double* sub_out,
                         double* cmin_out, double* cmax_out, cudaStream_t st, std::string* err) {
  using W = WarpCfg<D, P, SYS>;
  if (!W::GS && !set_smem(detect_kernel<D, P, SYS>, W::SMEM)) {
    *err = "limiter tile exceeds shared memory";
    return ADG_ERR_UNSUPPORTED;
  }
  const int64_t E = n_elements(g);
  const int64_t nb = (E + W::WPBX - 1) / W::WPBX;
  const int64_t cap = W::GS ? kScratchBlocks : 148 * 64;
  const unsigned grid = (unsigned)(nb < cap ? nb : cap);
  double* gs = nullptr;
  if (W::GS && !(gs = lim_scratch((size_t)grid * W::BLOCK_DBL * 8, err))) return ADG_ERR_CUDA;
  cudaMemsetAsync(count, 0, sizeof(int32_t), st);
  detect_kernel<D, P, SYS><<<grid, W::WPBX * 32, W::GS ? 0 : W::SMEM, st>>>(
      prev_sub, cmin, cmax, cand, pred_bad, lim_grid(g, gh), E, d0, eps, force, troubled, idx,
      count, sub_out, cmin_out, cmax_out, gs);
  return lerr(err);
}

template <int D, int P, int SYS>
static int launch_rescue(const adg_grid* g, const double* prev_sub, const int32_t* idx,
                         const int32_t* count, int32_t cmax, const double* dt,
                         const adg_subcell_ghosts* gh, double* u_out, int32_t* failed,
                         double* sub_next, double* cmin_next, double* cmax_next,
                         cudaStream_t st, std::string* err) {
  constexpr bool GS = LimDbl<D, P, SYS>::RESCUE > LimDbl<D, P, SYS>::LIM;
  const size_t sm = GS ? 0 : rescue_smem<D, P, SYS>();
  if (!GS && !set_smem(rescue_kernel<D, P, SYS, 0>, sm)) {
    *err = "limiter window exceeds shared memory";
    return ADG_ERR_UNSUPPORTED;
  }
  if (cmax <= 0) return ADG_OK;
  const unsigned grid = (unsigned)(GS && cmax > kScratchBlocks ? kScratchBlocks : cmax);
  double* gs = nullptr;
  if (GS && !(gs = lim_scratch((size_t)grid * LimDbl<D, P, SYS>::RESCUE * 8, err))) return ADG_ERR_CUDA;
  rescue_kernel<D, P, SYS, 0><<<grid, LimCfg<D, P, SYS>::NT, sm, st>>>(
      prev_sub, idx, count, lim_grid(g, gh), dt, u_out, failed, nullptr, nullptr, nullptr,
      sub_next, cmin_next, cmax_next, gs);
  return lerr(err);
}

template <int D, int P, int SYS>
static int launch_muscl_windows(const adg_grid* g, const double* windows, int64_t nwin,
                                const int32_t* count_dev, const double* dt, double* avg_out,
                                uint8_t* fail_each, cudaStream_t st, std::string* err) {
  constexpr bool GS = LimDbl<D, P, SYS>::RESCUE > LimDbl<D, P, SYS>::LIM;
  const size_t sm = GS ? 0 : rescue_smem<D, P, SYS>();
  if (!GS && !set_smem(rescue_kernel<D, P, SYS, 1>, sm)) {
    *err = "limiter window exceeds shared memory";
    return ADG_ERR_UNSUPPORTED;
  }
  if (nwin <= 0) return ADG_OK;
  const int64_t cap = GS ? kScratchBlocks : 65535 * 8;
  const unsigned grid = (unsigned)(nwin < cap ? nwin : cap);
  double* gs = nullptr;
  if (GS && !(gs = lim_scratch((size_t)grid * LimDbl<D, P, SYS>::RESCUE * 8, err))) return ADG_ERR_CUDA;
  LimGrid G = lim_grid(g);
  for (int j = 0; j < 3; ++j) G.h[j] = j < g->dim ? g->dx[j] : 1.0;   // dx = subcell widths here
  rescue_kernel<D, P, SYS, 1><<<grid, LimCfg<D, P, SYS>::NT, sm, st>>>(
      nullptr, nullptr, count_dev, G, dt, nullptr, nullptr, windows, avg_out, fail_each, nullptr,
      nullptr, nullptr, gs);
  return lerr(err);
}

template <int D, int P, int SYS>
static int launch_recover(const adg_grid* g, const double* ubar, double* out, cudaStream_t st,
                          std::string* err) {
  using C = LimCfg<D, P, SYS>;
  constexpr bool GS = LimDbl<D, P, SYS>::RECOVER > LimDbl<D, P, SYS>::LIM;
  const size_t sm = GS ? 0 : LimDbl<D, P, SYS>::RECOVER * 8;
  if (!GS && !set_smem(recover_kernel<D, P, SYS>, sm)) {
    *err = "limiter tile exceeds shared memory";
    return ADG_ERR_UNSUPPORTED;
  }
  const int64_t E = n_elements(g);
  const int64_t cap = GS ? kScratchBlocks : 65535 * 8;
  const unsigned grid = (unsigned)(E < cap ? E : cap);
  double* gs = nullptr;
  if (GS && !(gs = lim_scratch((size_t)grid * LimDbl<D, P, SYS>::RECOVER * 8, err))) return ADG_ERR_CUDA;
  recover_kernel<D, P, SYS><<<grid, C::NT, sm, st>>>(ubar, E, out, gs);
  return lerr(err);
}

template <int D, int P, int SYS>
static int launch_flatten_cells(const adg_grid* g, double* nodal, const double* averages,
                                int32_t* nflat, cudaStream_t st, std::string* err) {
  constexpr bool GS = LimDbl<D, P, SYS>::PROJ > LimDbl<D, P, SYS>::LIM;
  const size_t sm = GS ? 0 : proj_smem<D, P, SYS>();
  if (!GS && !set_smem(flatten_cells_kernel<D, P, SYS>, sm)) {
    *err = "limiter tile exceeds shared memory";
    return ADG_ERR_UNSUPPORTED;
  }
  const int64_t E = n_elements(g);
  const int64_t cap = GS ? kScratchBlocks : 65535 * 8;
  const unsigned grid = (unsigned)(E < cap ? E : cap);
  double* gs = nullptr;
  if (GS && !(gs = lim_scratch((size_t)grid * LimDbl<D, P, SYS>::PROJ * 8, err))) return ADG_ERR_CUDA;
  cudaMemsetAsync(nflat, 0, sizeof(int32_t), st);
  flatten_cells_kernel<D, P, SYS><<<grid, LimCfg<D, P, SYS>::NT, sm, st>>>(nodal, averages, E,
                                                                 g->gamma - 1.0, nflat, gs);
  return lerr(err);
}

template <int D, int P, int SYS>
static int launch_flatten(const adg_grid* g, double* u, int32_t* nflat, cudaStream_t st,
                          std::string* err) {
  constexpr bool GS = LimDbl<D, P, SYS>::PROJ > LimDbl<D, P, SYS>::LIM;
  const size_t sm = GS ? 0 : proj_smem<D, P, SYS>();
  if (!GS && !set_smem(flatten_ic_kernel<D, P, SYS>, sm)) {
    *err = "limiter tile exceeds shared memory";
    return ADG_ERR_UNSUPPORTED;
  }
  const int64_t E = n_elements(g);
  const int64_t cap = GS ? kScratchBlocks : 65535 * 8;
  const unsigned grid = (unsigned)(E < cap ? E : cap);
  double* gs = nullptr;
  if (GS && !(gs = lim_scratch((size_t)grid * LimDbl<D, P, SYS>::PROJ * 8, err))) return ADG_ERR_CUDA;
  cudaMemsetAsync(nflat, 0, sizeof(int32_t), st);
  flatten_ic_kernel<D, P, SYS><<<grid, LimCfg<D, P, SYS>::NT, sm, st>>>(u, E, g->gamma - 1.0, nflat, gs);
  return lerr(err);
}

int project_subcells(const adg_grid* g, const double* u, double* sub, double* cmin, double* cmax,
                     cudaStream_t st, std::string* err) {
  int rc = ADG_OK;
  ADG_LIM_SWITCH(launch_prep, g, u, sub, cmin, cmax, st, err);
  return rc;
}

int detect(const adg_grid* g, const double* prev_sub, const double* cmin, const double* cmax,
           const double* cand, const uint8_t* pred_bad, double delta0, double eps, int force_all,
           const adg_subcell_ghosts* gh, uint8_t* troubled, int32_t* idx, int32_t* count,
           double* sub_out, double* cmin_out, double* cmax_out, cudaStream_t st,
           std::string* err) {
  if (!lim_supported(g, gh, err)) return ADG_ERR_UNSUPPORTED;
  int rc = ADG_OK;
  ADG_LIM_SWITCH(launch_detect, g, prev_sub, cmin, cmax, cand, pred_bad, delta0, eps, force_all,
                 gh, troubled, idx, count, sub_out, cmin_out, cmax_out, st, err);
  return rc;
}

int rescue(const adg_grid* g, const double* prev_sub, const int32_t* idx,
           const int32_t* count_dev, int32_t count_max, const double* dt_dev,
           const adg_subcell_ghosts* gh, double* u_out, int32_t* failed, double* sub_next,
           double* cmin_next, double* cmax_next, cudaStream_t st, std::string* err) {
  if (!lim_supported(g, gh, err)) return ADG_ERR_UNSUPPORTED;
  int rc = ADG_OK;
  ADG_LIM_SWITCH(launch_rescue, g, prev_sub, idx, count_dev, count_max, dt_dev, gh, u_out, failed,
                 sub_next, cmin_next, cmax_next, st, err);
  return rc;
}

int muscl_windows(const adg_grid* g, const double* windows, int64_t nwin,
                  const int32_t* count_dev, const double* dt_dev, double* avg_out,
                  uint8_t* fail_each, cudaStream_t st, std::string* err) {
  int rc = ADG_OK;
  ADG_LIM_SWITCH(launch_muscl_windows, g, windows, nwin, count_dev, dt_dev, avg_out, fail_each, st,
                 err);
  return rc;
}

int recover_subcells(const adg_grid* g, const double* ubar, double* out, cudaStream_t st,
                     std::string* err) {
  int rc = ADG_OK;
  ADG_LIM_SWITCH(launch_recover, g, ubar, out, st, err);
  return rc;
}

int flatten_cells(const adg_grid* g, double* nodal, const double* averages, int32_t* nflat,
                  cudaStream_t st, std::string* err) {
  int rc = ADG_OK;
  ADG_LIM_SWITCH(launch_flatten_cells, g, nodal, averages, nflat, st, err);
  return rc;
}

int flatten_ic(const adg_grid* g, double* u, int32_t* nflat, cudaStream_t st, std::string* err) {
  int rc = ADG_OK;
  ADG_LIM_SWITCH(launch_flatten, g, u, nflat, st, err);
  return rc;
}

}  // namespace adg
