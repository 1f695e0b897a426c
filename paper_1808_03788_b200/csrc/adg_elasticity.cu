// adg_elasticity.cu -- the ADER-DG time step for the 2-D diffuse-interface
// linear elasticity plugin (reference systems.py:237-345,
// DiffuseInterfaceElasticity: m = 9, state (sxx, syy, sxy, avx, avy, alpha,
// lam, mu, rho), a pure nonconservative product B(q).grad q, no flux, no
// source; max |lambda| = c_p = sqrt((lam + 2 mu) / rho); admissible = finite).
//
// Same step structure and device buffers as the Euler / advection paths, so
// the drop-in driver runs it unchanged:
//  * predictor (predictor.py:74-191 with the NCP branch of _rhs_conservative):
//    a thread owns one spatial node; the element's space-time tile sits
//    time-major in shared memory, gradients are D/dx line contractions of q
//    itself, the rate is -ncp(q, grad q) and the new iterate accumulates in
//    registers slice by slice (q_new(t) = g0[t] u + dt sum_s gw[t][s] rate(s));
//    traces in the face kernels' owner-role order; the volume term
//    dt |Omega| w_node sum_t w_t (-ncp(q_t, grad q_t)) (corrector.py:141-177);
//  * face kernel (corrector.py:65-129): path-conservative fluctuations,
//    B integrated along the straight segment q- -> q+ with the 3-point
//    Gauss-Legendre rule (PATH_POINTS = 3), Rusanov dissipation masked on the
//    stationary fields (diss_mask); d_low and d_high are stored separately
//    (not antisymmetric for an NCP system), time-integrated, element-major;
//  * update (corrector.py:180-205) with the wave-speed / count / totals
//    epilogue of the other systems.
#include <algorithm>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

namespace el {
constexpr int M = 9;
constexpr int SXX = 0, SYY = 1, SXY = 2, AVX = 3, AVY = 4, ALPHA = 5, LAM = 6, MU = 7, RHO = 8;
constexpr double ALPHA_FLOOR = 1e-3;   // systems.py:13
// diss_mask (systems.py:258): no jump dissipation on alpha and the material
__device__ __forceinline__ double mask(int v) { return v < ALPHA ? 1.0 : 0.0; }

// systems.py:269-294 (ncp), the reference's operation order
__device__ __forceinline__ void ncp(const double* q, const double* gx, const double* gy,
                                    double* out) {
  const double a = fmax(q[ALPHA], ALPHA_FLOOR);
  const double lam = q[LAM], mu = q[MU], rho = q[RHO];
  const double vx = q[AVX] / a;
  const double vy = q[AVY] / a;
  const double dvx_dx = (gx[AVX] - vx * gx[ALPHA]) / a;
  const double dvy_dy = (gy[AVY] - vy * gy[ALPHA]) / a;
  const double dvx_dy = (gy[AVX] - vx * gy[ALPHA]) / a;
  const double dvy_dx = (gx[AVY] - vy * gx[ALPHA]) / a;
  out[SXX] = -(lam * (dvx_dx + dvy_dy) + 2.0 * mu * dvx_dx);
  out[SYY] = -(lam * (dvx_dx + dvy_dy) + 2.0 * mu * dvy_dy);
  out[SXY] = -mu * (dvx_dy + dvy_dx);
  out[AVX] = -((a * (gx[SXX] + gy[SXY]) + q[SXX] * gx[ALPHA]) + q[SXY] * gy[ALPHA]) / rho;
  out[AVY] = -((a * (gx[SXY] + gy[SYY]) + q[SXY] * gx[ALPHA]) + q[SYY] * gy[ALPHA]) / rho;
  out[ALPHA] = 0.0;
  out[LAM] = 0.0;
  out[MU] = 0.0;
  out[RHO] = 0.0;
}

// the nonzero entries of B(q).n (systems.py:296-322) for n = e_axis,
// accumulated with weight w into b[15] in the order
// SXX:(AVX,AVY,ALPHA) SYY:(AVX,AVY,ALPHA) SXY:(AVX,AVY,ALPHA)
// AVX:(SXX,SXY,ALPHA) AVY:(SXY,SYY,ALPHA)
__device__ __forceinline__ void ncp_matrix_acc(const double* q, int axis, double w, double* b) {
  const double nx = axis == 0 ? 1.0 : 0.0, ny = axis == 1 ? 1.0 : 0.0;
  const double a = fmax(q[ALPHA], ALPHA_FLOOR);
  const double lam = q[LAM], mu = q[MU], rho = q[RHO];
  const double vx = q[AVX] / a;
  const double vy = q[AVY] / a;
  const double lp2m = lam + 2.0 * mu;
  double e[15];
  e[0] = -lp2m * nx / a;
  e[1] = -lam * ny / a;
  e[2] = (lp2m * vx * nx + lam * vy * ny) / a;
  e[3] = -lam * nx / a;
  e[4] = -lp2m * ny / a;
  e[5] = (lam * vx * nx + lp2m * vy * ny) / a;
  e[6] = -mu * ny / a;
  e[7] = -mu * nx / a;
  e[8] = mu * (vx * ny + vy * nx) / a;
  e[9] = -a * nx / rho;
  e[10] = -a * ny / rho;
  e[11] = -(q[SXX] * nx + q[SXY] * ny) / rho;
  e[12] = -a * nx / rho;
  e[13] = -a * ny / rho;
  e[14] = -(q[SXY] * nx + q[SYY] * ny) / rho;
#pragma unroll
  for (int k = 0; k < 15; ++k) b[k] += w * e[k];
}

__device__ __forceinline__ double cp(const double* q) { return sqrt((q[LAM] + 2.0 * q[MU]) / q[RHO]); }

// the full 9 x 9 B(q).n for a general normal (systems.py:296-322), as a
// dense row-major matrix accumulated with weight w (path_integral_B)
__device__ __forceinline__ void ncp_matrix_dense_acc(const double* q, double nx, double ny,
                                                     double w, double* b) {
  const double a = fmax(q[ALPHA], ALPHA_FLOOR);
  const double lam = q[LAM], mu = q[MU], rho = q[RHO];
  const double vx = q[AVX] / a;
  const double vy = q[AVY] / a;
  const double lp2m = lam + 2.0 * mu;
  b[SXX * 9 + AVX] += w * (-lp2m * nx / a);
  b[SXX * 9 + AVY] += w * (-lam * ny / a);
  b[SXX * 9 + ALPHA] += w * ((lp2m * vx * nx + lam * vy * ny) / a);
  b[SYY * 9 + AVX] += w * (-lam * nx / a);
  b[SYY * 9 + AVY] += w * (-lp2m * ny / a);
  b[SYY * 9 + ALPHA] += w * ((lam * vx * nx + lp2m * vy * ny) / a);
  b[SXY * 9 + AVX] += w * (-mu * ny / a);
  b[SXY * 9 + AVY] += w * (-mu * nx / a);
  b[SXY * 9 + ALPHA] += w * (mu * (vx * ny + vy * nx) / a);
  b[AVX * 9 + SXX] += w * (-a * nx / rho);
  b[AVX * 9 + SXY] += w * (-a * ny / rho);
  b[AVX * 9 + ALPHA] += w * (-(q[SXX] * nx + q[SXY] * ny) / rho);
  b[AVY * 9 + SXY] += w * (-a * nx / rho);
  b[AVY * 9 + SYY] += w * (-a * ny / rho);
  b[AVY * 9 + ALPHA] += w * (-(q[SXY] * nx + q[SYY] * ny) / rho);
}
}  // namespace el

// Pointwise face terms of the module API (corrector.py:58-129) for state
// pairs [n][9] and a general normal: path_integral_B (3-point Gauss rule
// along q- -> q+), riemann_dminus (mode 0) or the face_fluxes pair (mode 1).
__global__ void el_points_kernel(const double* __restrict__ qm_all,
                                 const double* __restrict__ qp_all, int64_t n, double nx,
                                 double ny, int mode, double* __restrict__ out_a,
                                 double* __restrict__ out_b, double* __restrict__ bpath) {
  constexpr int M = el::M;
  const double r15 = sqrt(0.6);
  const double sn[3] = {0.5 - 0.5 * r15, 0.5, 0.5 + 0.5 * r15};
  const double sw[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double qm[M], qp[M], jump[M], b[M * M];
#pragma unroll
    for (int v = 0; v < M; ++v) {
      qm[v] = qm_all[i * M + v];
      qp[v] = qp_all[i * M + v];
      jump[v] = qp[v] - qm[v];
    }
#pragma unroll
    for (int k = 0; k < M * M; ++k) b[k] = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double psi[M];
#pragma unroll
      for (int v = 0; v < M; ++v) psi[v] = qm[v] + sn[k] * jump[v];
      el::ncp_matrix_dense_acc(psi, nx, ny, sw[k], b);
    }
    if (bpath) {
#pragma unroll
      for (int k = 0; k < M * M; ++k) bpath[i * M * M + k] = b[k];
    }
    if (mode < 0) continue;
    const double smax = nan_max(el::cp(qm), el::cp(qp));
#pragma unroll
    for (int r = 0; r < M; ++r) {
      double bj = 0.0;
#pragma unroll
      for (int c = 0; c < M; ++c) bj = fma(b[r * M + c], jump[c], bj);
      const double diss = ((0.5 * smax) * jump[r]) * el::mask(r);
      if (mode == 0) {
        out_a[i * M + r] = -diss + 0.5 * bj;
      } else {
        out_a[i * M + r] = (0.0 + 0.5 * bj) - diss;
        out_b[i * M + r] = (-0.0 + 0.5 * bj) + diss;
      }
    }
  }
}

int el_points(int64_t n, const double* normal, int mode, const double* qm, const double* qp,
              double* out_a, double* out_b, double* bpath, cudaStream_t st, std::string* err) {
  if (n <= 0) return ADG_OK;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, 148 * 16));
  el_points_kernel<<<(unsigned)blocks, 128, 0, st>>>(qm, qp, n, normal[0], normal[1], mode,
                                                      out_a, out_b, bpath);
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

template <int P>
struct ElCfg {
  static constexpr int M = el::M;
  static constexpr int PD = P * P;
  static constexpr int EPB = (128 / PD) > 0 ? (128 / PD) : 1;
  static constexpr int NT = ((EPB * PD + 31) / 32) * 32;
  static constexpr int TB = PD * M + ((PD * M) & 1);    // trace block (adg_trace_block)
  static constexpr int ELEM = P * PD * M + PD * M;     // time-major tile + startup staging
  static constexpr size_t SMEM = ((size_t)EPB * ELEM + 2 * NT + 4 * EPB) * 8;
};

struct ElArgs {
  const double* u;
  const double* dt;
  double* q_out;
  double* vol;
  double* traces;
  uint8_t* pred_bad;
  int32_t* sweeps;
  int64_t n_elem;
  double dx[2];
  double tol;
  int max_iter;
  int min_iter;
  double dd[2 * kMaxP * kMaxP];   // D / dx_dir, [dir][P][P]
};

// gradients at node (ni, nj) of a [node][M] field: g_dir = (D / dx_dir) along dir
template <int P>
__device__ __forceinline__ void el_grad(const double* __restrict__ W, const double* dd, int ni,
                                        int nj, double* gx, double* gy) {
  constexpr int M = el::M;
#pragma unroll
  for (int v = 0; v < M; ++v) gx[v] = gy[v] = 0.0;
#pragma unroll
  for (int l = 0; l < P; ++l) {
    const double cx = dd[ni * P + l], cy = dd[P * P + nj * P + l];
    const double* wx = W + (l * P + nj) * M;
    const double* wy = W + (ni * P + l) * M;
#pragma unroll
    for (int v = 0; v < M; ++v) {
      gx[v] = fma(cx, wx[v], gx[v]);
      gy[v] = fma(cy, wy[v], gy[v]);
    }
  }
}

template <int P>
__global__ void __launch_bounds__(ElCfg<P>::NT)
el_predict_kernel(const __grid_constant__ ElArgs a) {
  using C = ElCfg<P>;
  constexpr int M = el::M, PD = C::PD, EPB = C::EPB, NT = C::NT;
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double esm[];
  double* red = esm + (size_t)EPB * C::ELEM;          // [NT][2]
  int* fl = reinterpret_cast<int*>(red + 2 * NT);      // frozen / conv / nsw / ok per element
  const int tid = threadIdx.x;
  const bool lane_ok = tid < EPB * PD;
  const int elx = lane_ok ? tid / PD : EPB - 1;
  const int item = lane_ok ? tid - elx * PD : PD - 1;
  const int ni = item / P, nj = item % P;
  const double dt = *a.dt;
  const double cv = a.dx[0] * a.dx[1];
  const double wnode = T.weights[ni] * T.weights[nj];
  const int64_t ngroups = (a.n_elem + EPB - 1) / EPB;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t e = g * EPB + elx;
    const bool valid = lane_ok && e < a.n_elem;
    double* Q = esm + (size_t)elx * C::ELEM;   // [t][node][M]
    double* W = Q + P * PD * M;                // [node][M]
    int* frozen = fl + 4 * elx;
    __syncthreads();
    if (tid < EPB) {
      const bool ve = g * EPB + tid < a.n_elem;
      fl[4 * tid] = ve ? 0 : 1;
      fl[4 * tid + 1] = 0;
      fl[4 * tid + 2] = 0;
      fl[4 * tid + 3] = 1;
    }
    double uu[M];
#pragma unroll
    for (int v = 0; v < M; ++v) {
      uu[v] = valid ? a.u[((size_t)e * PD + item) * M + v] : 0.0;
      if (lane_ok) W[item * M + v] = uu[v];
    }
    __syncthreads();
    // startup guess (predictor.py:99-126) with L(w) = -ncp(w, grad w)
    double k1[M], k2[M];
    {
      double gx[M], gy[M], nc[M];
      el_grad<P>(W, a.dd, ni, nj, gx, gy);
      el::ncp(uu, gx, gy, nc);
#pragma unroll
      for (int v = 0; v < M; ++v) k1[v] = 0.0 - nc[v];
    }
    if (P >= 3) {
      __syncthreads();
      if (lane_ok) {
#pragma unroll
        for (int v = 0; v < M; ++v) W[item * M + v] = uu[v] + dt * k1[v];
      }
      __syncthreads();
      double w[M], gx[M], gy[M], nc[M];
#pragma unroll
      for (int v = 0; v < M; ++v) w[v] = W[item * M + v];
      el_grad<P>(W, a.dd, ni, nj, gx, gy);
      el::ncp(w, gx, gy, nc);
#pragma unroll
      for (int v = 0; v < M; ++v) k2[v] = 0.0 - nc[v];
    }
    __syncthreads();   // W readers done (Q is written below)
    if (lane_ok) {
#pragma unroll 1
      for (int t = 0; t < P; ++t) {
        const double s = T.nodes[t] * dt;
        const double c2 = 0.5 * s * s / dt;
#pragma unroll
        for (int v = 0; v < M; ++v)
          Q[(t * PD + item) * M + v] = P <= 2 ? uu[v] + s * k1[v]
                                              : uu[v] + s * k1[v] + c2 * (k2[v] - k1[v]);
      }
    }
    // Picard sweeps (predictor.py:135-191), per-element freezing
    int it = 0;
    for (; it < a.max_iter; ++it) {
      __syncthreads();   // Q complete; previous readers of red / flags done
      bool all = true;
      for (int ee = 0; ee < EPB; ++ee) all = all && fl[4 * ee];
      if (all) break;
      const bool work = valid && !frozen[0];
      double qn[P][M];
      if (work) {
#pragma unroll
        for (int t = 0; t < P; ++t)
#pragma unroll
          for (int v = 0; v < M; ++v) qn[t][v] = 0.0;
#pragma unroll 1
        for (int s = 0; s < P; ++s) {
          const double* Qs = Q + s * PD * M;
          double q[M], gx[M], gy[M], nc[M];
#pragma unroll
          for (int v = 0; v < M; ++v) q[v] = Qs[item * M + v];
          el_grad<P>(Qs, a.dd, ni, nj, gx, gy);
          el::ncp(q, gx, gy, nc);
#pragma unroll
          for (int t = 0; t < P; ++t) {
            const double gws = T.gw[t * P + s];
#pragma unroll
            for (int v = 0; v < M; ++v) qn[t][v] = fma(gws, 0.0 - nc[v], qn[t][v]);
          }
        }
      }
      __syncthreads();   // every thread has read the old tile
      double sd = 0.0, sq = 0.0;
      if (work) {
#pragma unroll
        for (int t = 0; t < P; ++t) {
          const double g0 = T.g0[t];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            const double qv = qn[t][v] * dt + g0 * uu[v];
            double* qo = Q + (t * PD + item) * M + v;
            const double dq = *qo - qv;
            sd = fma(dq, dq, sd);
            sq = fma(qv, qv, sq);
            *qo = qv;
          }
        }
      }
      red[2 * tid] = lane_ok ? sd : 0.0;
      red[2 * tid + 1] = lane_ok ? sq : 0.0;
      __syncthreads();
      if (tid < EPB && !fl[4 * tid]) {
        double s1 = 0.0, s2 = 0.0;
        for (int x = 0; x < PD; ++x) {
          s1 += red[2 * (tid * PD + x)];
          s2 += red[2 * (tid * PD + x) + 1];
        }
        const double res = T.k1_opnorm * sqrt(s1);
        const double scale = 1.0 + sqrt(s2);
        const int c = res <= a.tol * scale;
        fl[4 * tid + 1] = c;
        fl[4 * tid + 2] = it + 1;
        if (c && it + 1 >= a.min_iter) fl[4 * tid] = 1;
      }
    }
    __syncthreads();
    // admissibility (finite), traces, volume term, q_out
    if (valid) {
      bool ok = true;
      double sv[M];
#pragma unroll
      for (int v = 0; v < M; ++v) sv[v] = 0.0;
#pragma unroll 1
      for (int t = 0; t < P; ++t) {
        const double* Qt = Q + t * PD * M;
        double q[M], gx[M], gy[M], nc[M];
#pragma unroll
        for (int v = 0; v < M; ++v) {
          q[v] = Qt[item * M + v];
          ok = ok && isfinite(q[v]);
        }
        el_grad<P>(Qt, a.dd, ni, nj, gx, gy);
        el::ncp(q, gx, gy, nc);
#pragma unroll
        for (int v = 0; v < M; ++v) sv[v] = fma(T.weights[t], 0.0 - nc[v], sv[v]);
        if (a.q_out) {
#pragma unroll
          for (int v = 0; v < M; ++v) a.q_out[(((size_t)e * PD + item) * P + t) * M + v] = q[v];
        }
      }
      if (!ok) atomicAnd(&fl[4 * elx + 3], 0);
      // acc = dt |Omega| w_tensor sum_t w_t interior (corrector.py:166-168)
#pragma unroll
      for (int v = 0; v < M; ++v) a.vol[((size_t)e * PD + item) * M + v] = ((dt * cv) * wnode) * sv[v];
      // traces (face kernels' owner-role order: x [j][t], y [t][i]); this
      // thread's item is one line at one time for each direction
      const size_t fs = (size_t)a.n_elem * C::TB;
#pragma unroll
      for (int dir = 0; dir < 2; ++dir) {
        const int t = item % P, i0 = item / P;   // x: (j = i0, t); y: (t = item / P, i = item % P)
        const int tt = dir == 0 ? t : item / P;
        const int ii = dir == 0 ? i0 : item % P;
        double lo[M], hi[M];
#pragma unroll
        for (int v = 0; v < M; ++v) lo[v] = hi[v] = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          const int nd = dir == 0 ? l * P + ii : ii * P + l;
          const double* qv = Q + (tt * PD + nd) * M;
#pragma unroll
          for (int v = 0; v < M; ++v) {
            lo[v] = fma(T.left[l], qv[v], lo[v]);
            hi[v] = fma(T.right[l], qv[v], hi[v]);
          }
        }
        double* tlo = a.traces + (size_t)(2 * dir) * fs + (size_t)e * C::TB + (size_t)item * M;
#pragma unroll
        for (int v = 0; v < M; ++v) {
          tlo[v] = lo[v];
          tlo[fs + v] = hi[v];
        }
      }
    }
    __syncthreads();
    if (tid < EPB && g * EPB + tid < a.n_elem) {
      const int64_t ee = g * EPB + tid;
      a.pred_bad[ee] = (fl[4 * tid + 1] ? 0 : ADG_PRED_NOT_CONVERGED) | (fl[4 * tid + 3] ? 0 : ADG_PRED_INADMISSIBLE);
      a.sweeps[ee] = fl[4 * tid + 2] ? fl[4 * tid + 2] : it;
    }
  }
}

// Path-conservative Rusanov fluctuations (corrector.py:65-129): thread per
// (face, tangential node); d_low (minus element, its high face) and d_high
// (plus element, its low face), each sum_t w_t d_t, element-major
template <int P>
__global__ void el_face_kernel(const double* __restrict__ traces, double* __restrict__ fd,
                               int axis, int64_t c0, int64_t c1, int bc_lo, int bc_hi) {
  using C = ElCfg<P>;
  constexpr int M = el::M, PF = P, TB = C::TB;
  const DegreeTables& T = tab<P>();
  const int64_t n[2] = {c0, c1};
  int64_t nf[2] = {c0, c1};
  nf[axis] += 1;
  const int64_t faces = nf[0] * nf[1];
  const int64_t E = c0 * c1;
  const size_t fs = (size_t)E * TB;
  const double* tr_lo = traces + (size_t)(2 * axis) * fs;
  const double* tr_hi = tr_lo + fs;
  // 3-point Gauss-Legendre rule on [0, 1] (corrector.py:21-22)
  const double r15 = sqrt(0.6);
  const double sn[3] = {0.5 - 0.5 * r15, 0.5, 0.5 + 0.5 * r15};
  const double sw[3] = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < faces * PF;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = w / PF;
    const int tg = (int)(w - f * PF);
    int64_t c[2] = {f / nf[1], f % nf[1]};
    const int64_t fa = c[axis];
    auto eidx = [&](int64_t ca) {
      int64_t cc[2] = {c[0], c[1]};
      cc[axis] = ca;
      return cc[0] * n[1] + cc[1];
    };
    auto pos = [&](int t) { return axis == 0 ? tg * P + t : t * P + tg; };
    // face states (driver.py:234-261): periodic wrap; outflow copies the
    // interior trace; wall reflects it (systems.py:336-345)
    const double* pm;
    const double* pp;
    bool refl_m = false, refl_p = false;
    if (fa > 0) pm = tr_hi + (size_t)eidx(fa - 1) * TB;
    else if (bc_lo == ADG_BC_PERIODIC) pm = tr_hi + (size_t)eidx(n[axis] - 1) * TB;
    else { pm = tr_lo + (size_t)eidx(0) * TB; refl_m = bc_lo == ADG_BC_WALL; }
    if (fa < n[axis]) pp = tr_lo + (size_t)eidx(fa) * TB;
    else if (bc_hi == ADG_BC_PERIODIC) pp = tr_lo + (size_t)eidx(0) * TB;
    else { pp = tr_hi + (size_t)eidx(n[axis] - 1) * TB; refl_p = bc_hi == ADG_BC_WALL; }
    double dl[M], dh[M];
#pragma unroll
    for (int v = 0; v < M; ++v) dl[v] = dh[v] = 0.0;
#pragma unroll 1
    for (int t = 0; t < P; ++t) {
      double qm[M], qp[M], jump[M];
#pragma unroll
      for (int v = 0; v < M; ++v) {
        qm[v] = pm[pos(t) * M + v];
        qp[v] = pp[pos(t) * M + v];
      }
      // reflect (systems.py:336-345): normal stress components flip
      if (refl_m || refl_p) {
        double* q = refl_m ? qm : qp;
        if (axis == 0) { q[el::SXX] = -q[el::SXX]; q[el::SXY] = -q[el::SXY]; }
        else { q[el::SYY] = -q[el::SYY]; q[el::SXY] = -q[el::SXY]; }
      }
#pragma unroll
      for (int v = 0; v < M; ++v) jump[v] = qp[v] - qm[v];
      const double smax = nan_max(el::cp(qm), el::cp(qp));
      double b[15];
#pragma unroll
      for (int k = 0; k < 15; ++k) b[k] = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double psi[M];
#pragma unroll
        for (int v = 0; v < M; ++v) psi[v] = qm[v] + sn[k] * jump[v];
        el::ncp_matrix_acc(psi, axis, sw[k], b);
      }
      double bj[M];
      bj[el::SXX] = (b[0] * jump[el::AVX] + b[1] * jump[el::AVY]) + b[2] * jump[el::ALPHA];
      bj[el::SYY] = (b[3] * jump[el::AVX] + b[4] * jump[el::AVY]) + b[5] * jump[el::ALPHA];
      bj[el::SXY] = (b[6] * jump[el::AVX] + b[7] * jump[el::AVY]) + b[8] * jump[el::ALPHA];
      bj[el::AVX] = (b[9] * jump[el::SXX] + b[10] * jump[el::SXY]) + b[11] * jump[el::ALPHA];
      bj[el::AVY] = (b[12] * jump[el::SXY] + b[13] * jump[el::SYY]) + b[14] * jump[el::ALPHA];
      bj[el::ALPHA] = bj[el::LAM] = bj[el::MU] = bj[el::RHO] = 0.0;
      const double wt = T.weights[t];
#pragma unroll
      for (int v = 0; v < M; ++v) {
        const double diss = ((0.5 * smax) * jump[v]) * el::mask(v);
        const double half = 0.5 * bj[v];
        dl[v] = fma(wt, (0.0 + half) - diss, dl[v]);
        dh[v] = fma(wt, (-0.0 + half) + diss, dh[v]);
      }
    }
    // element-major [E][2 axes][2 sides][PF][M]
    if (fa > 0) {
      double* o = fd + (((size_t)eidx(fa - 1) * 2 + axis) * 2 + 1) * PF * M + (size_t)tg * M;
#pragma unroll
      for (int v = 0; v < M; ++v) o[v] = dl[v];
    }
    if (fa < n[axis]) {
      double* o = fd + (((size_t)eidx(fa) * 2 + axis) * 2 + 0) * PF * M + (size_t)tg * M;
#pragma unroll
      for (int v = 0; v < M; ++v) o[v] = dh[v];
    }
  }
}

// Per-node fold: wave speed c_p over admissible (finite) nodes, counts and
// the weighted conserved totals (driver.py:344-350)
__device__ __forceinline__ void el_node_fold(const double* q, double wnode, double& lam,
                                             unsigned& nadm, unsigned& nnf, double* tot) {
  constexpr int M = el::M;
  bool fin = true;
#pragma unroll
  for (int v = 0; v < M; ++v) fin = fin && isfinite(q[v]);
  nnf += fin ? 0u : 1u;
  if (fin) {
    ++nadm;
    lam = fmax(lam, el::cp(q));
  }
  if (tot) {
#pragma unroll
    for (int v = 0; v < M; ++v) tot[v] = fma(q[v], wnode, tot[v]);
  }
}

__device__ void el_block_fold(double lam, unsigned nadm, unsigned nnf, double* tot,
                              adg_reduce* red, double* partial) {
  constexpr int M = el::M, NW = kReduceThreads / 32;
  __shared__ double s_lam[NW];
  __shared__ unsigned s_cnt[NW][2];
  __shared__ double s_tot[NW][M];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, o));
  nadm = __reduce_add_sync(0xffffffffu, nadm);
  nnf = __reduce_add_sync(0xffffffffu, nnf);
#pragma unroll
  for (int v = 0; v < M; ++v) {
    double t = partial ? tot[v] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) s_tot[warp][v] = t;
  }
  if (lane == 0) {
    s_lam[warp] = lam;
    s_cnt[warp][0] = nadm;
    s_cnt[warp][1] = nnf;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double L = 0.0;
    unsigned long long na = 0, nn = 0;
    double Tt[M];
#pragma unroll
    for (int v = 0; v < M; ++v) Tt[v] = 0.0;
    for (int w = 0; w < NW; ++w) {
      L = fmax(L, s_lam[w]);
      na += s_cnt[w][0];
      nn += s_cnt[w][1];
#pragma unroll
      for (int v = 0; v < M; ++v) Tt[v] += s_tot[w][v];
    }
    if (red) {
      // c_p does not depend on the normal: the same speed on both axes
      atomic_max_pos(&red->lam_bits[0], L);
      atomic_max_pos(&red->lam_bits[1], L);
      if (na) atomicAdd(reinterpret_cast<unsigned long long*>(&red->n_admissible), na);
      if (nn) atomicAdd(reinterpret_cast<unsigned long long*>(&red->n_nonfinite), nn);
    }
    if (partial) {
#pragma unroll
      for (int v = 0; v < M; ++v) partial[(size_t)blockIdx.x * M + v] = Tt[v];
    }
  }
}

template <int P>
__global__ void __launch_bounds__(kReduceThreads)
el_reduce_kernel(const double* __restrict__ u, int64_t nodes, adg_reduce* red, double* partial) {
  constexpr int M = el::M, PD = P * P;
  const DegreeTables& T = tab<P>();
  double lam = 0.0, tot[M];
#pragma unroll
  for (int v = 0; v < M; ++v) tot[v] = 0.0;
  unsigned nadm = 0, nnf = 0;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int node = (int)(n % PD);
    el_node_fold(u + n * M, T.weights[node / P] * T.weights[node % P], lam, nadm, nnf,
                 partial ? tot : nullptr);
  }
  el_block_fold(lam, nadm, nnf, tot, red, partial);
}

// u* = u + (vol - acc_x,lo - acc_x,hi - acc_y,lo - acc_y,hi) / (|Omega| w_k)
// (corrector.py:180-205): face terms stored per side (d_high on the low face,
// d_low on the high face)
template <int P>
__global__ void __launch_bounds__(kReduceThreads)
el_update_kernel(const double* __restrict__ u, const double* __restrict__ vol,
                 const double* __restrict__ fd, const double* __restrict__ dt_dev,
                 double* __restrict__ u_out, int64_t E, double dx0, double dx1,
                 adg_reduce* red, double* partial) {
  constexpr int M = el::M, PD = P * P, PF = P;
  const DegreeTables& T = tab<P>();
  const double dt = *dt_dev;
  const double dx[2] = {dx0, dx1};
  const double cv = dx0 * dx1;
  double lam = 0.0, tot[M];
#pragma unroll
  for (int v = 0; v < M; ++v) tot[v] = 0.0;
  unsigned nadm = 0, nnf = 0;
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < E * PD;
       y += (int64_t)gridDim.x * blockDim.x) {
    const int64_t elx = y / PD;
    const int node = (int)(y - elx * PD);
    const int k[2] = {node / P, node % P};
    double total[M], q[M];
#pragma unroll
    for (int v = 0; v < M; ++v) total[v] = vol[y * M + v];
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
      const int tg = k[1 - ax];
      const double wtan = T.weights[tg];
      const double sc = dt * (cv / dx[ax]);
      const double* dlo = fd + (((size_t)elx * 2 + ax) * 2 + 0) * PF * M + (size_t)tg * M;
      const double* dhi = fd + (((size_t)elx * 2 + ax) * 2 + 1) * PF * M + (size_t)tg * M;
#pragma unroll
      for (int v = 0; v < M; ++v) total[v] -= sc * (T.left[k[ax]] * (dlo[v] * wtan));
#pragma unroll
      for (int v = 0; v < M; ++v) total[v] -= sc * (T.right[k[ax]] * (dhi[v] * wtan));
    }
    const double wnode = T.weights[k[0]] * T.weights[k[1]];
#pragma unroll
    for (int v = 0; v < M; ++v) {
      q[v] = u[y * M + v] + total[v] / (cv * wnode);
      u_out[y * M + v] = q[v];
    }
    el_node_fold(q, wnode, lam, nadm, nnf, partial ? tot : nullptr);
  }
  el_block_fold(lam, nadm, nnf, tot, red, partial);
}

__global__ void el_zero_reduce_kernel(adg_reduce* red) {
  if (threadIdx.x < sizeof(adg_reduce) / 8)
    reinterpret_cast<unsigned long long*>(red)[threadIdx.x] = 0ull;
}

// ------------------------------------------------------------------ launchers
#define ADG_EL_SWITCH(FN, ...)                                          \
  do {                                                                  \
    switch (g->degree + 1) {                                            \
      case 1: FN<1>(__VA_ARGS__); break;                                \
      case 2: FN<2>(__VA_ARGS__); break;                                \
      case 3: FN<3>(__VA_ARGS__); break;                                \
      case 4: FN<4>(__VA_ARGS__); break;                                \
      case 5: FN<5>(__VA_ARGS__); break;                                \
      case 6: FN<6>(__VA_ARGS__); break;                                \
      default:                                                          \
        *err = "elasticity-di on the device: degree <= 5";              \
        return ADG_ERR_UNSUPPORTED;                                     \
    }                                                                   \
  } while (0)

static int el_check(std::string* err) {
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

template <int P>
static void el_launch_predict(const ElArgs& a, int num_sms, cudaStream_t st) {
  using C = ElCfg<P>;
  static PerDevice attr;
  if (attr.first() && C::SMEM > 48 * 1024)
    cudaFuncSetAttribute(el_predict_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
  const int64_t ngroups = (a.n_elem + C::EPB - 1) / C::EPB;
  const int64_t grid = std::min<int64_t>(ngroups, (int64_t)num_sms * 16);
  if (grid > 0) el_predict_kernel<P><<<(unsigned)grid, C::NT, C::SMEM, st>>>(a);
}

int el_predict(const adg_grid* g, const double* u, const double* dt_dev, double tol,
               int max_iter, int min_iter, double* q_out, double* vol, double* traces,
               uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms,
               std::string* err) {
  ElArgs a{};
  a.u = u;
  a.dt = dt_dev;
  a.q_out = q_out;
  a.vol = vol;
  a.traces = traces;
  a.pred_bad = pred_bad;
  a.sweeps = sweeps;
  a.n_elem = n_elements(g);
  a.dx[0] = g->dx[0];
  a.dx[1] = g->dx[1];
  a.tol = tol;
  a.max_iter = max_iter > 0 ? max_iter : 2 * g->degree + 2;
  a.min_iter = min_iter;
  const int Pl = g->degree + 1;
  for (int dir = 0; dir < 2; ++dir)
    for (int x = 0; x < Pl * Pl; ++x) a.dd[dir * Pl * Pl + x] = h_tab[g->degree].diff[x] / g->dx[dir];
  ADG_EL_SWITCH(el_launch_predict, a, num_sms, st);
  return el_check(err);
}

template <int P>
static void el_launch_face(const adg_grid* g, int axis, const double* traces, double* fd,
                           cudaStream_t st) {
  int64_t nf[2] = {g->cells[0], g->cells[1]};
  nf[axis] += 1;
  const int64_t work = nf[0] * nf[1] * P;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((work + 127) / 128, 148 * 16));
  el_face_kernel<P><<<(unsigned)blocks, 128, 0, st>>>(traces, fd, axis, g->cells[0], g->cells[1],
                                                      g->bc[axis][0], g->bc[axis][1]);
}

int el_face_flux(const adg_grid* g, int axis, const double* traces, const double* ghost_lo,
                 const double* ghost_hi, double* fd, cudaStream_t st, std::string* err) {
  (void)ghost_lo;
  (void)ghost_hi;
  if (axis < 0 || axis >= 2) {
    *err = "axis out of range";
    return ADG_ERR_INVALID;
  }
  if (g->bc[axis][0] == ADG_BC_GHOST || g->bc[axis][1] == ADG_BC_GHOST) {
    *err = "elasticity-di on the device: exact / ghost faces are not supported";
    return ADG_ERR_UNSUPPORTED;
  }
  ADG_EL_SWITCH(el_launch_face, g, axis, traces, fd, st);
  return el_check(err);
}

template <int P>
static void el_launch_update(const adg_grid* g, const double* u, const double* vol,
                             const double* fd, const double* dt, double* u_out, adg_reduce* red,
                             double* partial, cudaStream_t st) {
  el_update_kernel<P><<<(unsigned)update_blocks(g), kReduceThreads, 0, st>>>(
      u, vol, fd, dt, u_out, n_elements(g), g->dx[0], g->dx[1], red, partial);
}

int el_update(const adg_grid* g, const double* u, const double* vol, const double* fd,
              const double* dt_dev, double* u_out, adg_reduce* red_next, double* partial,
              cudaStream_t st, std::string* err) {
  if (red_next) el_zero_reduce_kernel<<<1, 32, 0, st>>>(red_next);
  ADG_EL_SWITCH(el_launch_update, g, u, vol, fd, dt_dev, u_out, red_next, partial, st);
  return el_check(err);
}

template <int P>
static void el_launch_reduce(const adg_grid* g, const double* u, adg_reduce* red,
                             double* partial, cudaStream_t st) {
  el_reduce_kernel<P><<<(unsigned)reduce_blocks(g), kReduceThreads, 0, st>>>(
      u, n_elements(g) * P * P, red, partial);
}

int el_state_reduce(const adg_grid* g, const double* u, adg_reduce* red, double* partial,
                    cudaStream_t st, std::string* err) {
  if (red) el_zero_reduce_kernel<<<1, 32, 0, st>>>(red);
  ADG_EL_SWITCH(el_launch_reduce, g, u, red, partial, st);
  return el_check(err);
}

}  // namespace adg
