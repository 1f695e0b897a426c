// adg_advection.cu -- the ADER-DG time step for the scalar linear transport
// plugin q_t + a . grad q = 0 (reference systems.py:77-109, LinearAdvection:
// m = 1, F_j = a_j q, max |lambda| = |a . n|, admissible = finite).
//
// Same step structure and device buffers as the Euler path, so the drop-in
// driver runs it unchanged: a fused predictor (startup guess, Picard sweeps
// with per-element freezing, admissibility, face traces in the face kernels'
// owner-role block order, volume integral), a face kernel writing the
// time-integrated Rusanov terms element-major for both neighbours, and an
// update whose epilogue folds the next wave speeds, counts and fixed-order
// conserved-total partials.  With m = 1 a thread owns one spatial node at
// every time level (its P values in registers); line contractions read the
// neighbours' values from the element's time-major tile in shared memory.
#include <algorithm>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

template <int D, int P>
struct AdvCfg {
  static constexpr int PD = ipow(P, D);
  static constexpr int EPB = (256 / PD) > 0 ? (256 / PD) : 1;
  static constexpr int NT = ((EPB * PD + 31) / 32) * 32;
  static constexpr int TB = PD + (PD & 1);              // trace block (adg_trace_block)
  static constexpr int PF = PD / P;                      // tangential nodes per face
  // per element: time-major tile Q[t][node] + staged spatial field W[node] +
  // per-direction volume flux sums FB[dir][node]; + residual partials
  static constexpr int ELEM = P * PD + PD + D * PD;
  static constexpr size_t SMEM = ((size_t)EPB * ELEM + 2 * NT + 8 * EPB) * 8;
};

struct AdvArgs {
  const double* u;
  const double* q_init;   // optional starting iterate [E][P^d][P_t] (picard_solve initial=)
  const double* dt;
  double* q_out;
  double* vol;
  double* traces;
  uint8_t* pred_bad;
  int32_t* sweeps;
  int64_t n_elem;
  double dx[3];
  double a[3];
  double tol;
  int max_iter;
  int min_iter;
  double dd[3 * kMaxP * kMaxP];   // D / dx_dir, [dir][P][P]
};

template <int D, int P>
__device__ __forceinline__ int adv_node(int i, int j, int k) {
  return D == 3 ? (i * P + j) * P + k : (D == 2 ? i * P + j : i);
}

// L(w)(node) = ((0 - D_x (a_x w)) - D_y (a_y w)) - D_z (a_z w): the flux
// a_j w is formed first and contracted, x then y then z (predictor.py:86-90)
template <int D, int P>
__device__ __forceinline__ double adv_rate(const double* __restrict__ W, const double* dd,
                                           const double* a, int ni, int nj, int nk) {
  double r = 0.0;
#pragma unroll
  for (int dir = 0; dir < D; ++dir) {
    const int row = dir == 0 ? ni : (dir == 1 ? nj : nk);
    double y = 0.0;
#pragma unroll
    for (int l = 0; l < P; ++l) {
      const int nd = dir == 0 ? adv_node<D, P>(l, nj, nk)
                              : (dir == 1 ? adv_node<D, P>(ni, l, nk) : adv_node<D, P>(ni, nj, l));
      y = fma(dd[dir * P * P + row * P + l], a[dir] * W[nd], y);
    }
    r -= y;
  }
  return r;
}

template <int D, int P>
__global__ void __launch_bounds__(AdvCfg<D, P>::NT)
adv_predict_kernel(const __grid_constant__ AdvArgs a) {
  using C = AdvCfg<D, P>;
  constexpr int PD = C::PD, EPB = C::EPB, NT = C::NT;
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double asm_[];
  double* red = asm_ + (size_t)EPB * C::ELEM;          // [NT][2]
  int* fl = reinterpret_cast<int*>(red + 2 * NT);       // frozen / conv / nsw / ok per element
  const int tid = threadIdx.x;
  const bool lane_ok = tid < EPB * PD;
  const int el = lane_ok ? tid / PD : EPB - 1;
  const int item = lane_ok ? tid - el * PD : PD - 1;
  const int ni = D == 3 ? item / (P * P) : (D == 2 ? item / P : item);
  const int nj = D == 3 ? (item / P) % P : (D == 2 ? item % P : 0);
  const int nk = D == 3 ? item % P : 0;
  const double dt = *a.dt;
  const double av[3] = {a.a[0], a.a[1], a.a[2]};
  // volume scales (corrector.py:172-176, the reference's operation order)
  double vcoef[D];
  {
    const double cv = a.dx[0] * (D >= 2 ? a.dx[1] : 1.0) * (D == 3 ? a.dx[2] : 1.0);
    const double wnode = T.weights[ni] * (D >= 2 ? T.weights[nj] : 1.0) *
                         (D == 3 ? T.weights[nk] : 1.0);
#pragma unroll
    for (int dir = 0; dir < D; ++dir) {
      const int row = dir == 0 ? ni : (dir == 1 ? nj : nk);
      vcoef[dir] = (dt * cv / a.dx[dir]) * (wnode / T.weights[row]);
    }
  }
  const int64_t ngroups = (a.n_elem + EPB - 1) / EPB;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t e = g * EPB + el;
    const bool valid = lane_ok && e < a.n_elem;
    double* Q = asm_ + (size_t)el * C::ELEM;   // [t][node]
    double* W = Q + P * PD;                    // [node]
    double* FB = W + PD;                       // [dir][node]
    int* frozen = fl + 4 * el;
    __syncthreads();
    if (tid < EPB) {
      const bool ve = g * EPB + tid < a.n_elem;
      fl[4 * tid] = ve ? 0 : 1;
      fl[4 * tid + 1] = 0;
      fl[4 * tid + 2] = 0;
      fl[4 * tid + 3] = 1;
    }
    double uu = valid ? a.u[(size_t)e * PD + item] : 0.0;
    if (lane_ok) W[item] = uu;
    __syncthreads();
    // startup guess (predictor.py:99-126)
    double k1 = 0.0, k2 = 0.0;
    if (valid) k1 = adv_rate<D, P>(W, a.dd, av, ni, nj, nk);
    if (P >= 3) {
      __syncthreads();
      if (lane_ok) W[item] = uu + dt * k1;
      __syncthreads();
      if (valid) k2 = adv_rate<D, P>(W, a.dd, av, ni, nj, nk);
    }
    double q[P];
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const double s = T.nodes[t] * dt;
      if (P <= 2) q[t] = uu + s * k1;
      else {
        const double c2 = 0.5 * s * s / dt;
        q[t] = uu + s * k1 + c2 * (k2 - k1);
      }
      if (a.q_init && valid) q[t] = a.q_init[((size_t)e * PD + item) * P + t];
    }
    // Picard sweeps (predictor.py:135-191), per-element freezing
    int it = 0;
    for (; it < a.max_iter; ++it) {
      __syncthreads();   // previous readers of Q / red / flags are done
      bool all = true;
      for (int ee = 0; ee < EPB; ++ee) all = all && fl[4 * ee];
      if (all) break;
      const bool work = valid && !frozen[0];
      if (lane_ok) {
#pragma unroll
        for (int t = 0; t < P; ++t) Q[t * PD + item] = q[t];
      }
      __syncthreads();
      double sd = 0.0, sq = 0.0;
      if (work) {
        double r[P];
#pragma unroll
        for (int s = 0; s < P; ++s) r[s] = adv_rate<D, P>(Q + s * PD, a.dd, av, ni, nj, nk);
#pragma unroll
        for (int t = 0; t < P; ++t) {
          double c = 0.0;
#pragma unroll
          for (int s = 0; s < P; ++s) c = fma(T.gw[t * P + s], r[s], c);
          const double qn = c * dt + T.g0[t] * uu;
          const double dq = q[t] - qn;
          sd = fma(dq, dq, sd);
          sq = fma(qn, qn, sq);
          q[t] = qn;
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
    // admissibility (finite), final tile, traces, volume flux sums
    bool ok = true;
    if (lane_ok) {
#pragma unroll
      for (int t = 0; t < P; ++t) {
        ok = ok && isfinite(q[t]);
        Q[t * PD + item] = q[t];
      }
    }
    if (valid && !ok) fl[4 * el + 3] = 0;
    if (valid) {
#pragma unroll
      for (int dir = 0; dir < D; ++dir) {
        double f = 0.0;
#pragma unroll
        for (int t = 0; t < P; ++t) f = fma(T.weights[t], av[dir] * q[t], f);
        FB[dir * PD + item] = f;
      }
      if (a.q_out) {
#pragma unroll
        for (int t = 0; t < P; ++t) a.q_out[((size_t)e * PD + item) * P + t] = q[t];
      }
    }
    __syncthreads();
    if (valid) {
      // traces in the face kernels' owner-role block order (x: [j][k][t],
      // y: [k][t][i], z: [t][i][j]); this thread's item is one line at one t
      const size_t fs = (size_t)a.n_elem * C::TB;
#pragma unroll
      for (int dir = 0; dir < D; ++dir) {
        int t, i0, i1;
        if (D == 3) {
          if (dir == 0) { t = item % P; i0 = (item / P) % P; i1 = item / (P * P); }   // (t, k, j)
          else if (dir == 1) { i0 = item % P; t = (item / P) % P; i1 = item / (P * P); }
          else { i1 = item % P; i0 = (item / P) % P; t = item / (P * P); }
        } else if (D == 2) {
          if (dir == 0) { t = item % P; i0 = item / P; i1 = 0; }
          else { i0 = item % P; t = item / P; i1 = 0; }
        } else {
          t = item; i0 = 0; i1 = 0;
        }
        double lo = 0.0, hi = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          int nd;
          if (D == 3) nd = dir == 0 ? adv_node<D, P>(l, i1, i0)
                                    : (dir == 1 ? adv_node<D, P>(i0, l, i1) : adv_node<D, P>(i0, i1, l));
          else if (D == 2) nd = dir == 0 ? adv_node<D, P>(l, i0, 0) : adv_node<D, P>(i0, l, 0);
          else nd = l;
          const double qv = Q[t * PD + nd];
          lo = fma(T.left[l], qv, lo);
          hi = fma(T.right[l], qv, hi);
        }
        double* tlo = a.traces + (size_t)(2 * dir) * fs + (size_t)e * C::TB + item;
        tlo[0] = lo;
        tlo[fs] = hi;
      }
      // volume: contrib_dir = stiff x_dir fbar_dir, scaled and summed x, y, z
      double acc = 0.0;
#pragma unroll
      for (int dir = 0; dir < D; ++dir) {
        const int row = dir == 0 ? ni : (dir == 1 ? nj : nk);
        double y = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          const int nd = dir == 0 ? adv_node<D, P>(l, nj, nk)
                                  : (dir == 1 ? adv_node<D, P>(ni, l, nk) : adv_node<D, P>(ni, nj, l));
          y = fma(T.stiff[row * P + l], FB[dir * PD + nd], y);
        }
        acc += vcoef[dir] * y;
      }
      a.vol[(size_t)e * PD + item] = acc;
    }
    __syncthreads();
    if (tid < EPB && g * EPB + tid < a.n_elem) {
      const int64_t ee = g * EPB + tid;
      a.pred_bad[ee] = (fl[4 * tid + 1] ? 0 : ADG_PRED_NOT_CONVERGED) | (fl[4 * tid + 3] ? 0 : ADG_PRED_INADMISSIBLE);
      a.sweeps[ee] = fl[4 * tid + 2] ? fl[4 * tid + 2] : it;
    }
  }
}

// Rusanov face terms (corrector.py:100-129, :180-196): thread per (face,
// tangential node), time-integrated low-side term written element-major for
// the minus element's high face and the plus element's low face
template <int D, int P>
__global__ void adv_face_kernel(const double* __restrict__ traces, const double* __restrict__ ghost_lo,
                                const double* __restrict__ ghost_hi, double* __restrict__ fd,
                                int axis, int64_t c0, int64_t c1, int64_t c2, int bc_lo, int bc_hi,
                                double an) {
  using C = AdvCfg<D, P>;
  constexpr int PF = C::PF, TB = C::TB;
  const DegreeTables& T = tab<P>();
  const int64_t n[3] = {c0, c1, c2};
  int64_t nf[3] = {c0, c1, c2};
  nf[axis] += 1;
  const int64_t faces = nf[0] * (D >= 2 ? nf[1] : 1) * (D == 3 ? nf[2] : 1);
  const int64_t E = n[0] * (D >= 2 ? n[1] : 1) * (D == 3 ? n[2] : 1);
  const size_t fs = (size_t)E * TB;
  const double* tr_lo = traces + (size_t)(2 * axis) * fs;
  const double* tr_hi = tr_lo + fs;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < faces * PF;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = w / PF;
    const int tg = (int)(w - f * PF);
    int64_t c[3] = {0, 0, 0};
    {
      int64_t r = f;
      for (int j = D - 1; j >= 0; --j) {
        c[j] = r % nf[j];
        r /= nf[j];
      }
    }
    const int64_t fa = c[axis];
    auto eidx = [&](int64_t ca) {
      int64_t cc[3] = {c[0], c[1], c[2]};
      cc[axis] = ca;
      int64_t e = 0;
      for (int j = 0; j < D; ++j) e = e * n[j] + cc[j];
      return e;
    };
    // tangential index -> position inside a trace block (owner-role order)
    int a0 = 0, a1 = 0;
    if (D == 3) { a0 = tg / P; a1 = tg % P; }
    else if (D == 2) { a0 = tg; }
    auto pos = [&](int t) {
      if (D == 3) return axis == 0 ? (a0 * P + a1) * P + t
                                   : (axis == 1 ? (a1 * P + t) * P + a0 : (t * P + a0) * P + a1);
      if (D == 2) return axis == 0 ? a0 * P + t : t * P + a0;
      return t;
    };
    // face states (driver.py:234-261): minus = hi trace of element fa-1,
    // plus = lo trace of element fa; periodic wrap, the interior trace for
    // outflow and wall faces (a scalar's reflection is the identity,
    // systems.py base reflect), or the caller's exterior trace plane for
    // ghost ("exact") faces
    int64_t plane = 0;
    for (int j = 0; j < D; ++j)
      if (j != axis) plane = plane * n[j] + c[j];
    const double* pm;
    const double* pp;
    if (fa > 0) pm = tr_hi + (size_t)eidx(fa - 1) * TB;
    else if (bc_lo == ADG_BC_PERIODIC) pm = tr_hi + (size_t)eidx(n[axis] - 1) * TB;
    else if (bc_lo == ADG_BC_GHOST) pm = ghost_lo + (size_t)plane * TB;
    else pm = tr_lo + (size_t)eidx(0) * TB;
    if (fa < n[axis]) pp = tr_lo + (size_t)eidx(fa) * TB;
    else if (bc_hi == ADG_BC_PERIODIC) pp = tr_lo + (size_t)eidx(0) * TB;
    else if (bc_hi == ADG_BC_GHOST) pp = ghost_hi + (size_t)plane * TB;
    else pp = tr_hi + (size_t)eidx(n[axis] - 1) * TB;
    const double s = fabs(an);
    double dl = 0.0;
#pragma unroll
    for (int t = 0; t < P; ++t) {
      const double qm = pm[pos(t)], qp = pp[pos(t)];
      const double central = 0.5 * (an * qm + an * qp);
      const double diss = (0.5 * s) * (qp - qm);
      dl = fma(T.weights[t], (central + 0.0) - diss, dl);
    }
    if (fa > 0) fd[((size_t)eidx(fa - 1) * D + axis) * 2 * PF + PF + tg] = dl;
    if (fa < n[axis]) fd[((size_t)eidx(fa) * D + axis) * 2 * PF + tg] = dl;
  }
}

// Per-node wave speeds (|a_j| over finite nodes), counts and weighted totals
template <int D>
__device__ __forceinline__ void adv_node_fold(double q, const double* a, double wnode,
                                              double lam[3], unsigned& nadm, unsigned& nnf,
                                              double* tot) {
  const bool fin = isfinite(q);
  nnf += fin ? 0u : 1u;
  if (fin) {
    ++nadm;
#pragma unroll
    for (int j = 0; j < D; ++j) lam[j] = fmax(lam[j], fabs(a[j]));
  }
  if (tot) tot[0] = fma(q, wnode, tot[0]);
}

template <int D>
__device__ void adv_block_fold(double lam[3], unsigned nadm, unsigned nnf, const double* tot,
                               adg_reduce* red, double* partial) {
  constexpr int NW = kReduceThreads / 32;
  __shared__ double s_lam[NW][3];
  __shared__ unsigned s_cnt[NW][2];
  __shared__ double s_tot[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int j = 0; j < D; ++j) lam[j] = fmax(lam[j], __shfl_xor_sync(0xffffffffu, lam[j], o));
  }
  nadm = __reduce_add_sync(0xffffffffu, nadm);
  nnf = __reduce_add_sync(0xffffffffu, nnf);
  double t = partial ? tot[0] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < D; ++j) s_lam[warp][j] = lam[j];
    s_cnt[warp][0] = nadm;
    s_cnt[warp][1] = nnf;
    s_tot[warp] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double L[3] = {0.0, 0.0, 0.0};
    unsigned long long na = 0, nn = 0;
    double Tt = 0.0;
    for (int w = 0; w < NW; ++w) {
#pragma unroll
      for (int j = 0; j < D; ++j) L[j] = fmax(L[j], s_lam[w][j]);
      na += s_cnt[w][0];
      nn += s_cnt[w][1];
      Tt += s_tot[w];
    }
    if (red) {
#pragma unroll
      for (int j = 0; j < D; ++j) atomic_max_pos(&red->lam_bits[j], L[j]);
      if (na) atomicAdd(reinterpret_cast<unsigned long long*>(&red->n_admissible), na);
      if (nn) atomicAdd(reinterpret_cast<unsigned long long*>(&red->n_nonfinite), nn);
    }
    if (partial) partial[blockIdx.x] = Tt;
  }
}

template <int D, int P>
__device__ __forceinline__ double adv_weight(int node) {
  const DegreeTables& T = tab<P>();
  if (D == 1) return T.weights[node];
  if (D == 2) return T.weights[node / P] * T.weights[node % P];
  return T.weights[node / (P * P)] * T.weights[(node / P) % P] * T.weights[node % P];
}

template <int D, int P>
__global__ void __launch_bounds__(kReduceThreads)
adv_reduce_kernel(const double* __restrict__ u, int64_t nodes, double a0, double a1, double a2,
                  adg_reduce* red, double* partial) {
  constexpr int PD = ipow(P, D);
  const double av[3] = {a0, a1, a2};
  double lam[3] = {0.0, 0.0, 0.0};
  unsigned nadm = 0, nnf = 0;
  double tot = 0.0;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nodes;
       n += (int64_t)gridDim.x * blockDim.x)
    adv_node_fold<D>(u[n], av, adv_weight<D, P>((int)(n % PD)), lam, nadm, nnf,
                     partial ? &tot : nullptr);
  adv_block_fold<D>(lam, nadm, nnf, &tot, red, partial);
}

// u* = u + (vol - acc_x,lo - acc_x,hi - ...) / (|Omega| w_k)
// (corrector.py:180-205, the Euler update's operation order with m = 1)
template <int D, int P>
__global__ void __launch_bounds__(kReduceThreads)
adv_update_kernel(const double* __restrict__ u, const double* __restrict__ vol,
                  const double* __restrict__ fd, const double* __restrict__ dt_dev,
                  double* __restrict__ u_out, int64_t E, double dx0, double dx1, double dx2,
                  double a0, double a1, double a2, adg_reduce* red, double* partial) {
  constexpr int PD = ipow(P, D), PF = PD / P;
  const DegreeTables& T = tab<P>();
  const double dt = *dt_dev;
  const double dx[3] = {dx0, dx1, dx2};
  const double av[3] = {a0, a1, a2};
  const double cv = dx0 * (D >= 2 ? dx1 : 1.0) * (D == 3 ? dx2 : 1.0);
  double lam[3] = {0.0, 0.0, 0.0};
  unsigned nadm = 0, nnf = 0;
  double tot = 0.0;
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < E * PD;
       y += (int64_t)gridDim.x * blockDim.x) {
    const int64_t el = y / PD;
    const int node = (int)(y - el * PD);
    int k[3] = {0, 0, 0};
    if (D == 1) k[0] = node;
    if (D == 2) { k[0] = node / P; k[1] = node % P; }
    if (D == 3) { k[0] = node / (P * P); k[1] = (node / P) % P; k[2] = node % P; }
    double total = vol[y];
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      int tg = 0;
      double wtan = 1.0;
      bool first = true;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j == ax) continue;
        tg = tg * P + k[j];
        wtan = first ? T.weights[k[j]] : wtan * T.weights[k[j]];
        first = false;
      }
      const double sc = dt * (cv / dx[ax]);
      const double dlo = fd[((size_t)el * D + ax) * 2 * PF + tg];
      const double dhi = fd[((size_t)el * D + ax) * 2 * PF + PF + tg];
      const double blo = (D > 1) ? (-dlo) * wtan : -dlo;
      total -= sc * (T.left[k[ax]] * blo);
      const double bhi = (D > 1) ? dhi * wtan : dhi;
      total -= sc * (T.right[k[ax]] * bhi);
    }
    const double wnode = adv_weight<D, P>(node);
    const double q = u[y] + total / (cv * wnode);
    u_out[y] = q;
    adv_node_fold<D>(q, av, wnode, lam, nadm, nnf, partial ? &tot : nullptr);
  }
  adv_block_fold<D>(lam, nadm, nnf, &tot, red, partial);
}

__global__ void adv_zero_reduce_kernel(adg_reduce* red) {
  if (threadIdx.x < sizeof(adg_reduce) / 8)
    reinterpret_cast<unsigned long long*>(red)[threadIdx.x] = 0ull;
}

// ------------------------------------------------------------------ launchers
#define ADG_ADV_SWITCH(FN, ...)                                   \
  do {                                                            \
    switch (g->dim * 16 + g->degree + 1) {                        \
      case 17: FN<1, 1>(__VA_ARGS__); break;                      \
      case 18: FN<1, 2>(__VA_ARGS__); break;                      \
      case 19: FN<1, 3>(__VA_ARGS__); break;                      \
      case 20: FN<1, 4>(__VA_ARGS__); break;                      \
      case 21: FN<1, 5>(__VA_ARGS__); break;                      \
      case 22: FN<1, 6>(__VA_ARGS__); break;                      \
      case 23: FN<1, 7>(__VA_ARGS__); break;                      \
      case 24: FN<1, 8>(__VA_ARGS__); break;                      \
      case 25: FN<1, 9>(__VA_ARGS__); break;                      \
      case 26: FN<1, 10>(__VA_ARGS__); break;                     \
      case 33: FN<2, 1>(__VA_ARGS__); break;                      \
      case 34: FN<2, 2>(__VA_ARGS__); break;                      \
      case 35: FN<2, 3>(__VA_ARGS__); break;                      \
      case 36: FN<2, 4>(__VA_ARGS__); break;                      \
      case 37: FN<2, 5>(__VA_ARGS__); break;                      \
      case 38: FN<2, 6>(__VA_ARGS__); break;                      \
      case 39: FN<2, 7>(__VA_ARGS__); break;                      \
      case 40: FN<2, 8>(__VA_ARGS__); break;                      \
      case 41: FN<2, 9>(__VA_ARGS__); break;                      \
      case 42: FN<2, 10>(__VA_ARGS__); break;                     \
      case 49: FN<3, 1>(__VA_ARGS__); break;                      \
      case 50: FN<3, 2>(__VA_ARGS__); break;                      \
      case 51: FN<3, 3>(__VA_ARGS__); break;                      \
      case 52: FN<3, 4>(__VA_ARGS__); break;                      \
      case 53: FN<3, 5>(__VA_ARGS__); break;                      \
      case 54: FN<3, 6>(__VA_ARGS__); break;                      \
      default:                                                    \
        *err = "advection on the device: dim 1-2 any N, dim 3 N <= 5"; \
        return ADG_ERR_UNSUPPORTED;                               \
    }                                                             \
  } while (0)

static int adv_check(std::string* err) {
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

// L(q) = ((0 - D_x (a_x q)) - D_y (a_y q)) - .. at every node of a
// space-time q [E][P^d][P_t] (predictor.py:74-91 for m = 1); the
// weak_form_defect building block
template <int D, int P>
__global__ void __launch_bounds__(256)
adv_rate_kernel(const double* __restrict__ q, int64_t E, AdvArgs a, double* __restrict__ rate) {
  constexpr int PD = ipow(P, D);
  const int64_t total = E * PD * P;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = x / (PD * P);
    const int nd = (int)((x / P) % PD);
    const int t = (int)(x % P);
    const int ni = D == 3 ? nd / (P * P) : (D == 2 ? nd / P : nd);
    const int nj = D == 3 ? (nd / P) % P : (D == 2 ? nd % P : 0);
    const int nk = D == 3 ? nd % P : 0;
    double r = 0.0;
#pragma unroll
    for (int dir = 0; dir < D; ++dir) {
      const int row = dir == 0 ? ni : (dir == 1 ? nj : nk);
      double y = 0.0;
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const int n2 = dir == 0 ? adv_node<D, P>(l, nj, nk)
                                : (dir == 1 ? adv_node<D, P>(ni, l, nk) : adv_node<D, P>(ni, nj, l));
        y = fma(a.dd[dir * P * P + row * P + l], a.a[dir] * q[((size_t)e * PD + n2) * P + t], y);
      }
      r -= y;
    }
    rate[x] = r;
  }
}

template <int D, int P>
static void adv_launch_rate(const AdvArgs& a, const double* q, double* rate, cudaStream_t st) {
  const int64_t work = a.n_elem * ipow(P, D) * P;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 32));
  adv_rate_kernel<D, P><<<(unsigned)blocks, 256, 0, st>>>(q, a.n_elem, a, rate);
}

template <int D, int P>
static void adv_launch_predict(const AdvArgs& a, int num_sms, cudaStream_t st) {
  using C = AdvCfg<D, P>;
  static PerDevice attr;
  if (attr.first() && C::SMEM > 48 * 1024) {
    cudaFuncSetAttribute(adv_predict_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
  }
  const int64_t ngroups = (a.n_elem + C::EPB - 1) / C::EPB;
  const int64_t grid = std::min<int64_t>(ngroups, (int64_t)num_sms * 16);
  if (grid > 0) adv_predict_kernel<D, P><<<(unsigned)grid, C::NT, C::SMEM, st>>>(a);
}

int adv_predict(const adg_grid* g, const double* u, const double* dt_dev, double tol,
                int max_iter, int min_iter, double* q_out, double* vol, double* traces,
                uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms,
                std::string* err, const double* q_init, int startup_only) {
  AdvArgs a{};
  a.u = u;
  a.q_init = q_init;
  a.dt = dt_dev;
  a.q_out = q_out;
  a.vol = vol;
  a.traces = traces;
  a.pred_bad = pred_bad;
  a.sweeps = sweeps;
  a.n_elem = n_elements(g);
  for (int j = 0; j < 3; ++j) {
    a.dx[j] = j < g->dim ? g->dx[j] : 1.0;
    a.a[j] = j < g->dim ? g->velocity[j] : 0.0;
  }
  a.tol = tol;
  a.max_iter = startup_only ? 0 : (max_iter > 0 ? max_iter : 2 * g->degree + 2);
  a.min_iter = min_iter;
  const int Pl = g->degree + 1;
  for (int dir = 0; dir < 3; ++dir)
    for (int x = 0; x < Pl * Pl; ++x)
      a.dd[dir * Pl * Pl + x] = dir < g->dim ? h_tab[g->degree].diff[x] / g->dx[dir] : 0.0;
  ADG_ADV_SWITCH(adv_launch_predict, a, num_sms, st);
  return adv_check(err);
}

int adv_spacetime_rate(const adg_grid* g, const double* q, double* rate, cudaStream_t st,
                       std::string* err) {
  AdvArgs a{};
  a.n_elem = n_elements(g);
  for (int j = 0; j < 3; ++j) a.a[j] = j < g->dim ? g->velocity[j] : 0.0;
  const int Pl = g->degree + 1;
  for (int dir = 0; dir < 3; ++dir)
    for (int x = 0; x < Pl * Pl; ++x)
      a.dd[dir * Pl * Pl + x] = dir < g->dim ? h_tab[g->degree].diff[x] / g->dx[dir] : 0.0;
  if (a.n_elem == 0) return ADG_OK;
  ADG_ADV_SWITCH(adv_launch_rate, a, q, rate, st);
  return adv_check(err);
}

template <int D, int P>
static void adv_launch_face(const adg_grid* g, int axis, const double* traces,
                            const double* ghost_lo, const double* ghost_hi, double* fd,
                            cudaStream_t st) {
  int64_t nf[3] = {g->cells[0], D >= 2 ? g->cells[1] : 1, D == 3 ? g->cells[2] : 1};
  nf[axis] += 1;
  const int64_t work = nf[0] * nf[1] * nf[2] * (ipow(P, D) / P);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 16));
  adv_face_kernel<D, P><<<(unsigned)blocks, 256, 0, st>>>(
      traces, ghost_lo, ghost_hi, fd, axis, g->cells[0], D >= 2 ? g->cells[1] : 1,
      D == 3 ? g->cells[2] : 1, g->bc[axis][0], g->bc[axis][1], g->velocity[axis]);
}

int adv_face_flux(const adg_grid* g, int axis, const double* traces, const double* ghost_lo,
                  const double* ghost_hi, double* fd, cudaStream_t st, std::string* err) {
  if (axis < 0 || axis >= g->dim) {
    *err = "axis out of range";
    return ADG_ERR_INVALID;
  }
  if ((g->bc[axis][0] == ADG_BC_GHOST && !ghost_lo) ||
      (g->bc[axis][1] == ADG_BC_GHOST && !ghost_hi)) {
    *err = "ghost boundary without ghost traces";
    return ADG_ERR_UNSUPPORTED;
  }
  ADG_ADV_SWITCH(adv_launch_face, g, axis, traces, ghost_lo, ghost_hi, fd, st);
  return adv_check(err);
}

template <int D, int P>
static void adv_launch_update(const adg_grid* g, const double* u, const double* vol,
                              const double* fd, const double* dt, double* u_out,
                              adg_reduce* red, double* partial, cudaStream_t st) {
  adv_update_kernel<D, P><<<(unsigned)update_blocks(g), kReduceThreads, 0, st>>>(
      u, vol, fd, dt, u_out, n_elements(g), g->dx[0], D >= 2 ? g->dx[1] : 1.0,
      D == 3 ? g->dx[2] : 1.0, g->velocity[0], g->velocity[1], g->velocity[2], red, partial);
}

int adv_update(const adg_grid* g, const double* u, const double* vol, const double* fd,
               const double* dt_dev, double* u_out, adg_reduce* red_next, double* partial,
               cudaStream_t st, std::string* err) {
  if (red_next) adv_zero_reduce_kernel<<<1, 32, 0, st>>>(red_next);
  ADG_ADV_SWITCH(adv_launch_update, g, u, vol, fd, dt_dev, u_out, red_next, partial, st);
  return adv_check(err);
}

template <int D, int P>
static void adv_launch_reduce(const adg_grid* g, const double* u, adg_reduce* red,
                              double* partial, cudaStream_t st) {
  adv_reduce_kernel<D, P><<<(unsigned)reduce_blocks(g), kReduceThreads, 0, st>>>(
      u, n_elements(g) * ipow(P, D), g->velocity[0], g->velocity[1], g->velocity[2], red,
      partial);
}

int adv_state_reduce(const adg_grid* g, const double* u, adg_reduce* red, double* partial,
                     cudaStream_t st, std::string* err) {
  if (red) adv_zero_reduce_kernel<<<1, 32, 0, st>>>(red);
  ADG_ADV_SWITCH(adv_launch_reduce, g, u, red, partial, st);
  return adv_check(err);
}

}  // namespace adg
