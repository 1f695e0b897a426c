// adg_predictor.cu -- fused element-local ADER-DG predictor for sm_100a.
//
// One launch does, per element: the startup guess (predictor.py:99-126),
// the space-time Picard fixed point (predictor.py:135-191), the final
// admissibility screen (predictor.py:188-189), face-trace extraction
// (predictor.py:218-230) and the corrector's volume integral
// (corrector.py:141-177).  The space-time tile of an element never leaves
// the SM (shared memory; an L2-resident global slab for the 3-D N>=6
// tiles that exceed 227 KB).  HBM traffic is u in, vol + traces out.
//
// Work decomposition of one Picard sweep (P = N+1 nodes per axis, m vars):
//  phase 1  "line" role: a thread owns one x-line of the tile at one time
//           node, evaluates the Euler flux on its P nodes, contracts the
//           x-flux with D_x in registers, and publishes F_y (F_z) planes;
//  phase 2  same thread adds the y (z) derivative of its line from the
//           published planes (lanes sharing a plane read it by broadcast);
//  phase 3  "node" role: a thread owns one spatial node at all P time
//           nodes, applies the time operator gw (registers), forms
//           q_new = dt * gw.rate + g0 u and the residual partials.
// Residual norms are reduced per element in a fixed order (bitwise
// deterministic); an element freezes at its first converged sweep
// (>= min_iter).  SURVEY.md Appendix A: per-element stopping differs from
// the reference's global rule by <= 1e-14.
#include <algorithm>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

template <int D, int P>
struct PredCfg {
  static constexpr int M = D + 2;
  static constexpr int PD = ipow(P, D);      // spatial nodes
  static constexpr int PT = PD * P;          // space-time nodes
  static constexpr int TILE = PT * M;        // doubles in one space-time tile
  // flux planes exchanged between line threads: F_y (D>=2) and F_z (D=3),
  // stored with the contraction index fastest and padded to an even count
  // so a thread reads two nodes per 128-bit shared load
  static constexpr int NF = (D == 3) ? 2 : (D == 2 ? 1 : 0);
  static constexpr int PL = P + (P & 1);
  static constexpr int PLANE = PD * M * PL;  // doubles per exchanged flux buffer
  static constexpr int FREG_A = NF * PLANE;
  static constexpr int FREG_B = D * PD * M;
  static constexpr int FREG_AB = FREG_A > FREG_B ? FREG_A : FREG_B;
  static constexpr int FREG = FREG_AB > TILE ? FREG_AB : TILE;  // also holds the rate
  static constexpr int TILE_PAD = TILE + (TILE & 1);   // keeps F 16-byte aligned
  static constexpr int ELEM = TILE_PAD + FREG + (FREG & 1);   // doubles per element slab
  static constexpr int BUDGET = 110 * 1024;  // bytes of tiles per CTA (>= 2 CTAs/SM)
  static constexpr int EPB_T = (256 / PD) > 0 ? (256 / PD) : 1;
  static constexpr int EPB_S = (BUDGET / (ELEM * 8)) > 0 ? (BUDGET / (ELEM * 8)) : 1;
  static constexpr int EPB = EPB_T < EPB_S ? EPB_T : EPB_S;
  static constexpr int NT = ((EPB * PD + 31) / 32) * 32;
  static constexpr int NW = NT / 32;
  // small shared data: scaled D (3 P^2), reduction partials (2 NT), flags
  static constexpr int SMALL_DBL = ((3 * P * P + 2 * NT + 1) / 2) * 2;
  static constexpr int FLAGS = 5 * EPB + 1;
  static constexpr size_t SMALL_BYTES = SMALL_DBL * 8 + ((FLAGS * 4 + 15) / 16) * 16;
  static constexpr size_t TILE_BYTES = (size_t)EPB * ELEM * 8;
  static constexpr bool SMEM_TILES = (SMALL_BYTES + TILE_BYTES) <= 220 * 1024;
  static constexpr size_t SMEM_BYTES = SMALL_BYTES + (SMEM_TILES ? TILE_BYTES : 0);
};

struct PredArgs {
  const double* u;
  const double* dt;
  double* q_out;
  double* vol;
  double* traces;
  uint8_t* pred_bad;
  int32_t* sweeps;
  double* ws;          // global tile workspace (large-tile variant)
  int64_t n_elem;
  double dx[3];
  double gamma;
  double tol;
  int max_iter;
  int min_iter;
};

// index of a space-time tile value: [node][t][v]
template <int P, int M>
__device__ __forceinline__ int qi(int node, int t, int v) {
  return (node * P + t) * M + v;
}

// spatial node index from per-axis indices (row-major, last axis fastest)
template <int D, int P>
__device__ __forceinline__ int node3(int i, int j, int k) {
  if (D == 3) return (i * P + j) * P + k;
  if (D == 2) return i * P + j;
  return i;
}

// exchanged flux planes: F_y plane (i, k, t) and F_z plane (i, j, t), each
// holding v-rows of PL contiguous values along the contraction axis
template <int D, int P>
__device__ __forceinline__ int fy_idx(int i, int k, int t, int v) {
  constexpr int M = D + 2, PL = P + (P & 1);
  return D == 3 ? (((i * P + k) * P + t) * M + v) * PL : ((i * P + t) * M + v) * PL;
}
template <int P>
__device__ __forceinline__ int fz_idx(int i, int j, int t, int v) {
  constexpr int M = 5, PL = P + (P & 1);
  return (((i * P + j) * P + t) * M + v) * PL;
}

// L(w) = -sum_j (D/dx_j) F_j(w) at one node from published per-node fluxes
// F[(dir*PD + node)*M + v]; accumulated x then y then z (predictor.py:86-90).
template <int D, int P>
__device__ __forceinline__ void node_rate(const double* __restrict__ F, const double* Ds, int i,
                                          int j, int k, double out[D + 2]) {
  using C = PredCfg<D, P>;
  constexpr int M = C::M, PD = C::PD;
#pragma unroll
  for (int v = 0; v < M; ++v) out[v] = 0.0;
#pragma unroll
  for (int dir = 0; dir < D; ++dir) {
    const int row = dir == 0 ? i : (dir == 1 ? j : k);
    double acc[M];
#pragma unroll
    for (int v = 0; v < M; ++v) acc[v] = 0.0;
#pragma unroll
    for (int l = 0; l < P; ++l) {
      const int nd = dir == 0 ? node3<D, P>(l, j, k)
                              : (dir == 1 ? node3<D, P>(i, l, k) : node3<D, P>(i, j, l));
      const double dl = Ds[dir * P * P + row * P + l];
#pragma unroll
      for (int v = 0; v < M; ++v) acc[v] = fma(dl, F[(dir * PD + nd) * M + v], acc[v]);
    }
#pragma unroll
    for (int v = 0; v < M; ++v) out[v] -= acc[v];
  }
}

template <int D, int P>
__global__ void __launch_bounds__(PredCfg<D, P>::NT)
predict_kernel(PredArgs a) {
  using C = PredCfg<D, P>;
  constexpr int M = C::M, PD = C::PD, TILE = C::TILE, EPB = C::EPB, NT = C::NT;
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double smem[];
  double* Ds = smem;                          // [3][P][P] D / dx_dir
  double* red = Ds + 3 * P * P;               // [NT][2]
  int* fl = reinterpret_cast<int*>(red + 2 * NT);
  int* frozen = fl;                           // [EPB]
  int* conv = fl + EPB;                       // [EPB]
  int* nsw = fl + 2 * EPB;                    // [EPB]
  int* okf = fl + 3 * EPB;                    // [EPB]
  int* valid_e = fl + 4 * EPB;                // [EPB]
  int* all_frozen = fl + 5 * EPB;
  double* tiles;
  if constexpr (C::SMEM_TILES) {
    tiles = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + C::SMALL_BYTES);
  } else {
    tiles = a.ws + (size_t)blockIdx.x * EPB * C::ELEM;
  }

  const int tid = threadIdx.x;
  const int el = tid / PD;
  const int item = tid - el * PD;
  const bool lane_ok = el < EPB;
  const double gm1 = a.gamma - 1.0;
  const double dt = *a.dt;
  const int max_iter = a.max_iter;

  for (int x = tid; x < D * P * P; x += NT) {
    const int dir = x / (P * P);
    const double h = dir == 0 ? a.dx[0] : (dir == 1 ? a.dx[1] : a.dx[2]);
    Ds[x] = T.diff[x - dir * P * P] / h;
  }

  // node-role coordinates
  const int ni = (D == 3) ? item / (P * P) : (D == 2 ? item / P : item);
  const int nj = (D == 3) ? (item / P) % P : (D == 2 ? item % P : 0);
  const int nk = (D == 3) ? item % P : 0;
  // line-role coordinates: x-line (la, lb) at time lt, la fastest so that
  // the P lanes reading one F_y plane (same lb, lt) sit in one warp and the
  // shared loads broadcast
  const int la = (D >= 2) ? item % P : 0;
  const int lb = (D == 3) ? (item / P) % P : 0;
  const int lt = (D == 3) ? item / (P * P) : (D == 2 ? item / P : item);

  const int64_t ngroups = (a.n_elem + EPB - 1) / EPB;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t e = g * EPB + el;
    const bool valid = lane_ok && e < a.n_elem;
    double* Q = tiles + (lane_ok ? el : 0) * C::ELEM;
    double* F = Q + C::TILE_PAD;
    __syncthreads();  // Ds ready / previous group finished with the tiles
    if (tid < EPB) {
      const bool ve = g * EPB + tid < a.n_elem;
      valid_e[tid] = ve;
      frozen[tid] = ve ? 0 : 1;
      conv[tid] = 0;
      nsw[tid] = 0;
      okf[tid] = 1;
    }
    if (tid == 0) *all_frozen = 0;

    // ---------------- startup guess (node role) ----------------------
    double uu[M];
    double k1[M];
    if (valid) {
      const double* ue = a.u + (size_t)e * PD * M + (size_t)item * M;
#pragma unroll
      for (int v = 0; v < M; ++v) uu[v] = ue[v];
      double f[D][M];
      flux_all<D>(uu, gm1, f);
#pragma unroll
      for (int dir = 0; dir < D; ++dir)
#pragma unroll
        for (int v = 0; v < M; ++v) F[(dir * PD + item) * M + v] = f[dir][v];
    }
    __syncthreads();
    if (valid) node_rate<D, P>(F, Ds, ni, nj, nk, k1);
    double k2[M];
    if (P >= 3) {
      __syncthreads();
      if (valid) {
        double w[M];
#pragma unroll
        for (int v = 0; v < M; ++v) w[v] = uu[v] + dt * k1[v];
        double f[D][M];
        flux_all<D>(w, gm1, f);
#pragma unroll
        for (int dir = 0; dir < D; ++dir)
#pragma unroll
          for (int v = 0; v < M; ++v) F[(dir * PD + item) * M + v] = f[dir][v];
      }
      __syncthreads();
      if (valid) node_rate<D, P>(F, Ds, ni, nj, nk, k2);
    }
    if (valid) {
#pragma unroll
      for (int t = 0; t < P; ++t) {
        const double s = T.nodes[t] * dt;
        if (P <= 2) {
#pragma unroll
          for (int v = 0; v < M; ++v) Q[qi<P, M>(item, t, v)] = uu[v] + s * k1[v];
        } else {
          const double c2 = 0.5 * s * s / dt;
#pragma unroll
          for (int v = 0; v < M; ++v)
            Q[qi<P, M>(item, t, v)] = uu[v] + s * k1[v] + c2 * (k2[v] - k1[v]);
        }
      }
    }
    __syncthreads();

    // ---------------- Picard sweeps -----------------------------------
    int it = 0;
    for (; it < max_iter; ++it) {
      if (*all_frozen) break;
      const bool work = valid && !frozen[el];
      double rate[P][M];
      // phase 1: line role, x contraction in registers, publish F_y/F_z
      if (work) {
        double ql[P][M];
#pragma unroll
        for (int l = 0; l < P; ++l)
#pragma unroll
          for (int v = 0; v < M; ++v) ql[l][v] = Q[qi<P, M>(node3<D, P>(l, la, lb), lt, v)];
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
          for (int v = 0; v < M; ++v) rate[i][v] = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          double f[D][M];
          flux_all<D>(ql[l], gm1, f);
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const double dil = Ds[i * P + l];
#pragma unroll
            for (int v = 0; v < M; ++v) rate[i][v] = fma(dil, f[0][v], rate[i][v]);
          }
          // F_y at node (l, la, lb, lt) -> plane (i=l, k=lb, t=lt), slot j=la
          if (D >= 2) {
#pragma unroll
            for (int v = 0; v < M; ++v) F[fy_idx<D, P>(l, lb, lt, v) + la] = f[1][v];
          }
          // F_z -> plane (i=l, j=la, t=lt), slot k=lb
          if (D == 3) {
#pragma unroll
            for (int v = 0; v < M; ++v) F[C::PLANE + fz_idx<P>(l, la, lt, v) + lb] = f[2][v];
          }
        }
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
          for (int v = 0; v < M; ++v) rate[i][v] = -rate[i][v];
      }
      if (D >= 2) {
        __syncthreads();
        // phase 2: y (and z) derivatives of the owned line; the P lanes of a
        // warp that share a plane read it by broadcast, two nodes per load
        if (work) {
          double dr[C::PL];
#pragma unroll
          for (int l = 0; l < C::PL; ++l) dr[l] = l < P ? Ds[P * P + la * P + l] : 0.0;
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int v = 0; v < M; ++v) {
              const double2* row =
                  reinterpret_cast<const double2*>(F + fy_idx<D, P>(i, lb, lt, v));
              double s = 0.0;
#pragma unroll
              for (int l2 = 0; l2 < C::PL / 2; ++l2) {
                const double2 fv = row[l2];
                s = fma(dr[2 * l2], fv.x, s);
                if (2 * l2 + 1 < P) s = fma(dr[2 * l2 + 1], fv.y, s);
              }
              rate[i][v] -= s;
            }
          if (D == 3) {
#pragma unroll
            for (int l = 0; l < C::PL; ++l) dr[l] = l < P ? Ds[2 * P * P + lb * P + l] : 0.0;
#pragma unroll
            for (int i = 0; i < P; ++i)
#pragma unroll
              for (int v = 0; v < M; ++v) {
                const double2* row =
                    reinterpret_cast<const double2*>(F + C::PLANE + fz_idx<P>(i, la, lt, v));
                double s = 0.0;
#pragma unroll
                for (int l2 = 0; l2 < C::PL / 2; ++l2) {
                  const double2 fv = row[l2];
                  s = fma(dr[2 * l2], fv.x, s);
                  if (2 * l2 + 1 < P) s = fma(dr[2 * l2 + 1], fv.y, s);
                }
                rate[i][v] -= s;
              }
          }
        }
      }
      __syncthreads();
      // phase 2b: publish the rate (reuses the F_y plane)
      if (work) {
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
          for (int v = 0; v < M; ++v) F[qi<P, M>(node3<D, P>(i, la, lb), lt, v)] = rate[i][v];
      }
      __syncthreads();
      // phase 3: node role, time operator + residual
      double sd = 0.0, sq = 0.0;
      if (work) {
        double r[P][M];
#pragma unroll
        for (int s = 0; s < P; ++s)
#pragma unroll
          for (int v = 0; v < M; ++v) r[s][v] = F[qi<P, M>(item, s, v)];
#pragma unroll
        for (int t = 0; t < P; ++t) {
          const double g0 = T.g0[t];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            double c = 0.0;
#pragma unroll
            for (int s = 0; s < P; ++s) c = fma(T.gw[t * P + s], r[s][v], c);
            const double qn = c * dt + g0 * uu[v];
            const double dq = Q[qi<P, M>(item, t, v)] - qn;
            sd = fma(dq, dq, sd);
            sq = fma(qn, qn, sq);
            Q[qi<P, M>(item, t, v)] = qn;
          }
        }
      }
      red[2 * tid] = sd;
      red[2 * tid + 1] = sq;
      __syncthreads();
      // per-element fixed-order reduction; warp w handles elements w, w+NW, ..
      {
        const int warp = tid >> 5, lane = tid & 31;
        for (int ee = warp; ee < EPB; ee += C::NW) {
          double s1 = 0.0, s2 = 0.0;
          for (int x = lane; x < PD; x += 32) {
            s1 += red[2 * (ee * PD + x)];
            s2 += red[2 * (ee * PD + x) + 1];
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
          }
          if (lane == 0 && !frozen[ee]) {
            const double res = T.k1_opnorm * sqrt(s1);
            const double scale = 1.0 + sqrt(s2);
            const int c = res <= a.tol * scale;
            conv[ee] = c;
            nsw[ee] = it + 1;
            if (c && it + 1 >= a.min_iter) frozen[ee] = 1;
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        int all = 1;
        for (int ee = 0; ee < EPB; ++ee) all &= frozen[ee];
        *all_frozen = all;
      }
      __syncthreads();
    }

    // ---------------- admissibility of the converged tile --------------
    if (valid) {
      bool ok = true;
#pragma unroll
      for (int t = 0; t < P; ++t) {
        double q[M];
#pragma unroll
        for (int v = 0; v < M; ++v) q[v] = Q[qi<P, M>(item, t, v)];
        ok = ok && admissible<D>(q, gm1);
      }
      if (!ok) okf[el] = 0;
    }

    // ---------------- traces (line role) ------------------------------
    if (valid) {
      const size_t face_stride = (size_t)a.n_elem * PD * M;
      const size_t eoff = (size_t)e * PD * M;
      const int tang = (D == 3) ? (la * P + lb) : (D == 2 ? la : 0);
#pragma unroll
      for (int dir = 0; dir < D; ++dir) {
        double lo[M], hi[M];
#pragma unroll
        for (int v = 0; v < M; ++v) lo[v] = hi[v] = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          const int nd = dir == 0 ? node3<D, P>(l, la, lb)
                                  : (dir == 1 ? node3<D, P>(la, l, lb) : node3<D, P>(la, lb, l));
          const double pl = T.left[l], pr = T.right[l];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            const double qv = Q[qi<P, M>(nd, lt, v)];
            lo[v] = fma(pl, qv, lo[v]);
            hi[v] = fma(pr, qv, hi[v]);
          }
        }
        double* tlo = a.traces + (size_t)(2 * dir) * face_stride + eoff + (size_t)(tang * P + lt) * M;
        double* thi = tlo + face_stride;
#pragma unroll
        for (int v = 0; v < M; ++v) {
          tlo[v] = lo[v];
          thi[v] = hi[v];
        }
      }
      if (a.q_out) {
        double* qo = a.q_out + (size_t)e * TILE + (size_t)item * P * M;
#pragma unroll
        for (int x = 0; x < P * M; ++x) qo[x] = Q[item * P * M + x];
      }
    }
    // ---------------- volume integral (node role) ----------------------
    // fbar_j = sum_t w_t F_j(q_t) (corrector.py:171), published per node
    __syncthreads();  // F region free (rate no longer needed)
    if (valid) {
      double fb[D][M];
#pragma unroll
      for (int dir = 0; dir < D; ++dir)
#pragma unroll
        for (int v = 0; v < M; ++v) fb[dir][v] = 0.0;
#pragma unroll
      for (int t = 0; t < P; ++t) {
        double q[M];
#pragma unroll
        for (int v = 0; v < M; ++v) q[v] = Q[qi<P, M>(item, t, v)];
        double f[D][M];
        flux_all<D>(q, gm1, f);
        const double wt = T.weights[t];
#pragma unroll
        for (int dir = 0; dir < D; ++dir)
#pragma unroll
          for (int v = 0; v < M; ++v) fb[dir][v] = fma(wt, f[dir][v], fb[dir][v]);
      }
#pragma unroll
      for (int dir = 0; dir < D; ++dir)
#pragma unroll
        for (int v = 0; v < M; ++v) F[(dir * PD + item) * M + v] = fb[dir][v];
    }
    __syncthreads();
    if (valid) {
      const double cv = a.dx[0] * (D >= 2 ? a.dx[1] : 1.0) * (D == 3 ? a.dx[2] : 1.0);
      const double wnode = T.weights[ni] * (D >= 2 ? T.weights[nj] : 1.0) *
                           (D == 3 ? T.weights[nk] : 1.0);
      double acc[M];
#pragma unroll
      for (int v = 0; v < M; ++v) acc[v] = 0.0;
#pragma unroll
      for (int dir = 0; dir < D; ++dir) {
        const int row = dir == 0 ? ni : (dir == 1 ? nj : nk);
        const double coef = (dt * cv / a.dx[dir]) * (wnode / T.weights[row]);
        double c[M];
#pragma unroll
        for (int v = 0; v < M; ++v) c[v] = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          const int nd = dir == 0 ? node3<D, P>(l, nj, nk)
                                  : (dir == 1 ? node3<D, P>(ni, l, nk) : node3<D, P>(ni, nj, l));
          const double sl = T.stiff[row * P + l];
#pragma unroll
          for (int v = 0; v < M; ++v) c[v] = fma(sl, F[(dir * PD + nd) * M + v], c[v]);
        }
#pragma unroll
        for (int v = 0; v < M; ++v) acc[v] += coef * c[v];
      }
      double* vo = a.vol + (size_t)e * PD * M + (size_t)item * M;
#pragma unroll
      for (int v = 0; v < M; ++v) vo[v] = acc[v];
    }
    __syncthreads();
    if (tid < EPB && valid_e[tid]) {
      const int64_t ee = g * EPB + tid;
      a.pred_bad[ee] = !(conv[tid] && okf[tid]);
      a.sweeps[ee] = nsw[tid] ? nsw[tid] : it;
    }
  }
}

template <int D, int P>
static int launch_predict(const PredArgs& a0, cudaStream_t st, int num_sms, double* ws_pool,
                          size_t ws_bytes, std::string* err) {
  using C = PredCfg<D, P>;
  auto kern = predict_kernel<D, P>;
  static bool attr_set = false;
  if (!attr_set) {
    if (C::SMEM_BYTES > 48 * 1024) {
      cudaError_t ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)C::SMEM_BYTES);
      if (ce != cudaSuccess) {
        *err = cudaGetErrorString(ce);
        return ADG_ERR_CUDA;
      }
    }
    attr_set = true;
  }
  PredArgs a = a0;
  const int64_t ngroups = (a.n_elem + C::EPB - 1) / C::EPB;
  int64_t grid;
  if (C::SMEM_TILES) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NT, C::SMEM_BYTES);
    if (per_sm < 1) per_sm = 1;
    grid = std::min<int64_t>(ngroups, (int64_t)num_sms * per_sm * 8);
  } else {
    const size_t per_cta = (size_t)C::EPB * C::ELEM * 8;
    int64_t cap = (int64_t)(ws_bytes / per_cta);
    grid = std::min<int64_t>(ngroups, std::min<int64_t>(cap, (int64_t)num_sms * 2));
    if (grid < 1) {
      *err = "predictor workspace too small";
      return ADG_ERR_RUNTIME;
    }
    a.ws = ws_pool;
  }
  if (grid < 1) return ADG_OK;
  kern<<<(unsigned)grid, C::NT, C::SMEM_BYTES, st>>>(a);
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

template <int D, int P>
static size_t ws_need(int num_sms) {
  using C = PredCfg<D, P>;
  return C::SMEM_TILES ? 0 : (size_t)C::EPB * C::ELEM * 8 * num_sms * 2;
}

#define ADG_DISPATCH_P(D, FN, ...)                       \
  switch (P) {                                           \
    case 1: return FN<D, 1>(__VA_ARGS__);                \
    case 2: return FN<D, 2>(__VA_ARGS__);                \
    case 3: return FN<D, 3>(__VA_ARGS__);                \
    case 4: return FN<D, 4>(__VA_ARGS__);                \
    case 5: return FN<D, 5>(__VA_ARGS__);                \
    case 6: return FN<D, 6>(__VA_ARGS__);                \
    case 7: return FN<D, 7>(__VA_ARGS__);                \
    case 8: return FN<D, 8>(__VA_ARGS__);                \
    case 9: return FN<D, 9>(__VA_ARGS__);                \
    case 10: return FN<D, 10>(__VA_ARGS__);              \
  }

size_t predict_workspace_bytes(int dim, int P, int num_sms) {
  if (dim == 1) { ADG_DISPATCH_P(1, ws_need, num_sms) }
  if (dim == 2) { ADG_DISPATCH_P(2, ws_need, num_sms) }
  if (dim == 3) { ADG_DISPATCH_P(3, ws_need, num_sms) }
  return 0;
}

int predict(const adg_grid* g, const double* u, const double* dt_dev, double tol, int max_iter,
            int min_iter, double* q_out, double* vol, double* traces, uint8_t* pred_bad,
            int32_t* sweeps, cudaStream_t st, int num_sms, double* ws, size_t ws_bytes,
            std::string* err) {
  PredArgs a{};
  a.u = u;
  a.dt = dt_dev;
  a.q_out = q_out;
  a.vol = vol;
  a.traces = traces;
  a.pred_bad = pred_bad;
  a.sweeps = sweeps;
  a.ws = nullptr;
  a.n_elem = g->cells[0] * (g->dim >= 2 ? g->cells[1] : 1) * (g->dim == 3 ? g->cells[2] : 1);
  for (int j = 0; j < 3; ++j) a.dx[j] = j < g->dim ? g->dx[j] : 1.0;
  a.gamma = g->gamma;
  a.tol = tol;
  a.max_iter = max_iter > 0 ? max_iter : 2 * g->degree + 2;
  a.min_iter = min_iter;
  const int P = g->degree + 1;
  if (g->dim == 1) { ADG_DISPATCH_P(1, launch_predict, a, st, num_sms, ws, ws_bytes, err) }
  if (g->dim == 2) { ADG_DISPATCH_P(2, launch_predict, a, st, num_sms, ws, ws_bytes, err) }
  if (g->dim == 3) { ADG_DISPATCH_P(3, launch_predict, a, st, num_sms, ws, ws_bytes, err) }
  *err = "unsupported dim/degree";
  return ADG_ERR_UNSUPPORTED;
}

}  // namespace adg
