// adg_pieces.cu -- the reference's corrector module functions as standalone
// device calls (sm_100a), for callers that use the module API directly
// instead of Simulation (SURVEY.md §8(b) "module functions"):
//   face_fluxes     (corrector.py:100-129)  pointwise Rusanov pair
//   volume_integral (corrector.py:141-177)  from a given space-time q
//   face_integral   (corrector.py:180-196)  one face's accumulator
//   element_update  (corrector.py:199-205)  u + (vol - sum faces) / mass
//   extract_traces  (predictor.py:218-230)  face states of a given q
//   space-time rate (predictor.py:74-91, :94-96)  L(q) at every node (the
//                   weak_form_defect check of predictor.py:194-215)
// The fused time step (adg_predict / adg_face_flux / adg_update) does not
// use these; they trade fusion for the reference's array interfaces.
// Arrays are in the reference layouts with the element grid flattened to E.
#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

namespace {

constexpr int kPieceThreads = 256;

template <int D>
__global__ void __launch_bounds__(kPieceThreads)
face_points_kernel(const double* __restrict__ qm, const double* __restrict__ qp, int64_t n,
                   int axis, double gamma, double* __restrict__ dlow,
                   double* __restrict__ dhigh) {
  constexpr int M = D + 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[M], b[M], lo[M], hi[M];
#pragma unroll
    for (int v = 0; v < M; ++v) {
      a[v] = qm[i * M + v];
      b[v] = qp[i * M + v];
    }
    rusanov_pair<D>(a, b, axis, gamma, gamma - 1.0, lo, hi);
#pragma unroll
    for (int v = 0; v < M; ++v) {
      dlow[i * M + v] = lo[v];
      dhigh[i * M + v] = hi[v];
    }
  }
}

// One-sided Rusanov term for a general outward normal (riemann_dminus,
// corrector.py:81-97): -1/2 s (q+ - q-) + sum_j 1/2 n_j (F_j(q-) + F_j(q+)),
// s = max(|lambda(q-).n|, |lambda(q+).n|).  SYS 0: Euler (m = D + 2);
// SYS 1: advection (m = 1, F_j = a_j q).  MODE 1 forms the face_fluxes pair
// (corrector.py:100-129) for n = e_axis instead.
template <int SYS, int D>
__global__ void __launch_bounds__(kPieceThreads)
riemann_points_kernel(const double* __restrict__ qm_all, const double* __restrict__ qp_all,
                      int64_t n, double n0, double n1, double n2, double gamma, double a0,
                      double a1, double a2, int mode, double* __restrict__ out_a,
                      double* __restrict__ out_b) {
  constexpr int M = SYS == 0 ? D + 2 : 1;
  const double nv[3] = {n0, n1, n2};
  const double av[3] = {a0, a1, a2};
  const double gm1 = gamma - 1.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double qm[M], qp[M];
#pragma unroll
    for (int v = 0; v < M; ++v) {
      qm[v] = qm_all[i * M + v];
      qp[v] = qp_all[i * M + v];
    }
    double s;
    if (SYS == 0) {
      double um = 0.0, up = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        um = um + qm[1 + j] * nv[j];
        up = up + qp[1 + j] * nv[j];
      }
      const double lm = fabs(um / qm[0]) + sqrt(gamma * pressure<D>(qm, gm1) / qm[0]);
      const double lp = fabs(up / qp[0]) + sqrt(gamma * pressure<D>(qp, gm1) / qp[0]);
      s = nan_max(lm, lp);
    } else {
      double an = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) an = an + av[j] * nv[j];
      s = fabs(an);
    }
    if (mode == 2) {   // rusanov_theta (corrector.py:58-62): the speed alone, [n]
      out_a[i] = s;
      continue;
    }
    double out[M], fm[M], fp[M];
#pragma unroll
    for (int v = 0; v < M; ++v) out[v] = -0.5 * s * (qp[v] - qm[v]);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (nv[j] == 0.0) continue;
      if (SYS == 0) {
        flux_axis<D>(qm, gm1, j, fm);
        flux_axis<D>(qp, gm1, j, fp);
      } else {
        fm[0] = av[j] * qm[0];
        fp[0] = av[j] * qp[0];
      }
      if (mode == 1) {
        // face pair along e_j (only one nonzero component)
#pragma unroll
        for (int v = 0; v < M; ++v) {
          const double central = 0.5 * (fm[v] + fp[v]);
          const double diss = 0.5 * s * (qp[v] - qm[v]);
          out_a[i * M + v] = (central + 0.0) - diss;
          out_b[i * M + v] = (-central + 0.0) + diss;
        }
        break;
      }
#pragma unroll
      for (int v = 0; v < M; ++v) out[v] += 0.5 * nv[j] * (fm[v] + fp[v]);
    }
    if (mode == 0) {
#pragma unroll
      for (int v = 0; v < M; ++v) out_a[i * M + v] = out[v];
    }
  }
}


// ---- limiter module pieces (limiter.py:45-101), array interfaces ----------
// minmod (limiter.py:45-48): the smaller-magnitude argument where the signs
// agree, else 0
__global__ void __launch_bounds__(kPieceThreads)
minmod_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
              double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[i], y = b[i];
    const double pick = fabs(x) <= fabs(y) ? x : y;
    out[i] = x * y > 0.0 ? pick : 0.0;
  }
}

// per-cell extrema of a subcell field [ncell][nsub][m] (NaN propagates like
// numpy's amin / amax)
__global__ void __launch_bounds__(kPieceThreads)
cell_extrema_kernel(const double* __restrict__ x, int64_t ncell, int nsub, int m,
                    double* __restrict__ cmin, double* __restrict__ cmax) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncell * m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / m;
    const int v = (int)(i - c * m);
    const double* p = x + c * nsub * m + v;
    double lo = p[0], hi = p[0];
    for (int s = 1; s < nsub; ++s) {
      const double q = p[(int64_t)s * m];
      lo = (q < lo || q != q) ? q : lo;
      hi = (q > hi || q != q) ? q : hi;
    }
    cmin[i] = lo;
    cmax[i] = hi;
  }
}

// relaxed DMP bounds (limiter.py:51-73) of the core cells of a one-cell
// padded grid: own and 2 d face-neighbour extrema, widened by
// max(delta0, eps (hi - lo))
__global__ void __launch_bounds__(kPieceThreads)
relaxed_bounds_kernel(const double* __restrict__ cmin, const double* __restrict__ cmax, int dim,
                      int64_t n0, int64_t n1, int64_t n2, int m, double delta0, double eps,
                      double* __restrict__ lo_out, double* __restrict__ hi_out) {
  const int64_t n[3] = {n0, n1, n2};
  const int64_t ncore = n0 * (dim >= 2 ? n1 : 1) * (dim == 3 ? n2 : 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncore * m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / m;
    const int v = (int)(i - c * m);
    int64_t k[3] = {0, 0, 0}, r = c;
    for (int j = dim - 1; j >= 0; --j) {
      k[j] = r % n[j];
      r /= n[j];
    }
    auto padded = [&](const int64_t* kk) {
      int64_t idx = 0;
      for (int j = 0; j < dim; ++j) idx = idx * (n[j] + 2) + (kk[j] + 1);
      return idx * m + v;
    };
    double lo = cmin[padded(k)], hi = cmax[padded(k)];
    for (int j = 0; j < dim; ++j)
      for (int sh = -1; sh <= 1; sh += 2) {
        int64_t kk[3] = {k[0], k[1], k[2]};
        kk[j] += sh;
        const double a = cmin[padded(kk)], b = cmax[padded(kk)];
        lo = (a < lo || a != a) ? a : lo;      // torch.minimum / maximum: NaN propagates
        hi = (b > hi || b != b) ? b : hi;
      }
    const double w = eps * (hi - lo);
    const double delta = w != w ? w : (w < delta0 ? delta0 : w);   // clamp(min=delta0)
    lo_out[i] = lo - delta;
    hi_out[i] = hi + delta;
  }
}

// detect_troubled (limiter.py:76-86): a subcell outside the bounds, or an
// inadmissible nodal or subcell state.  SYS 0: Euler; SYS 1: finite only
// (advection, elasticity-di)
template <int SYS, int D>
__global__ void __launch_bounds__(kPieceThreads)
detect_cells_kernel(const double* __restrict__ cand, const double* __restrict__ sub,
                    const double* __restrict__ lo, const double* __restrict__ hi, int64_t E,
                    int pd, int sd, int m, double gm1, uint8_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    bool bad = false;
    auto adm = [&](const double* q) {
      if (SYS == 0) return admissible<D>(q, gm1);
      bool fin = true;
      for (int v = 0; v < m; ++v) fin = fin && isfinite(q[v]);
      return fin;
    };
    for (int s = 0; s < sd; ++s) {
      const double* q = sub + (e * sd + s) * m;
      for (int v = 0; v < m; ++v) bad = bad || q[v] < lo[e * m + v] || q[v] > hi[e * m + v];
      bad = bad || !adm(q);
    }
    for (int nd = 0; nd < pd; ++nd) bad = bad || !adm(cand + (e * pd + nd) * m);
    out[e] = bad ? 1 : 0;
  }
}

// gather_windows (limiter.py:89-101): out[w][a..][v] = padded[start_w + a][v]
__global__ void __launch_bounds__(kPieceThreads)
gather_windows_kernel(const double* __restrict__ padded, int dim, int64_t d0, int64_t d1,
                      int64_t d2, int m, const int64_t* __restrict__ starts, int64_t nwin,
                      int size, double* __restrict__ out) {
  const int64_t dims[3] = {d0, d1, d2};
  int64_t per = m;
  for (int j = 0; j < dim; ++j) per *= size;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nwin * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = i / per;
    int64_t r = i - w * per;
    const int v = (int)(r % m);
    r /= m;
    int64_t a[3] = {0, 0, 0};
    for (int j = dim - 1; j >= 0; --j) {
      a[j] = r % size;
      r /= size;
    }
    int64_t idx = 0;
    for (int j = 0; j < dim; ++j) idx = idx * dims[j] + (starts[w * dim + j] + a[j]);
    out[i] = padded[idx * m + v];
  }
}

// one CTA per element: node threads form fbar_dir = sum_t w_t F_dir(q_t),
// then the stiffness contraction per direction (corrector.py:167-176)
template <int D, int P>
__global__ void __launch_bounds__(kPieceThreads)
volume_kernel(const double* __restrict__ q, int64_t E, double dx0, double dx1, double dx2,
              double gamma, const double* __restrict__ dt_dev, double* __restrict__ vol) {
  constexpr int M = D + 2, PD = ipow(P, D);
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double fb[];   // [D][PD][M]
  const double dx[3] = {dx0, dx1, dx2};
  const double gm1 = gamma - 1.0;
  const double dt = *dt_dev;
  const double cv = dx0 * (D >= 2 ? dx1 : 1.0) * (D == 3 ? dx2 : 1.0);
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    for (int nd = threadIdx.x; nd < PD; nd += blockDim.x) {
      double acc[D][M];
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int v = 0; v < M; ++v) acc[j][v] = 0.0;
      for (int t = 0; t < P; ++t) {
        double f[D][M];
        flux_all<D>(q + (((size_t)e * PD + nd) * P + t) * M, gm1, f);
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
          for (int v = 0; v < M; ++v) acc[j][v] = fma(T.weights[t], f[j][v], acc[j][v]);
      }
#pragma unroll
      for (int j = 0; j < D; ++j)
#pragma unroll
        for (int v = 0; v < M; ++v) fb[(j * PD + nd) * M + v] = acc[j][v];
    }
    __syncthreads();
    for (int nd = threadIdx.x; nd < PD; nd += blockDim.x) {
      const int k[3] = {D == 3 ? nd / (P * P) : (D == 2 ? nd / P : nd),
                        D == 3 ? (nd / P) % P : (D == 2 ? nd % P : 0), D == 3 ? nd % P : 0};
      double wnode = T.weights[k[0]];
      if (D >= 2) wnode *= T.weights[k[1]];
      if (D == 3) wnode *= T.weights[k[2]];
      double out[M];
#pragma unroll
      for (int v = 0; v < M; ++v) out[v] = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const int stride = D == 3 ? (j == 0 ? P * P : (j == 1 ? P : 1)) : (D == 2 ? (j == 0 ? P : 1) : 1);
        const int base = nd - k[j] * stride;
        const double coef = (dt * cv / dx[j]) * (wnode / T.weights[k[j]]);
#pragma unroll
        for (int v = 0; v < M; ++v) {
          double c = 0.0;
          for (int l = 0; l < P; ++l)
            c = fma(T.stiff[k[j] * P + l], fb[(j * PD + base + l * stride) * M + v], c);
          out[v] += coef * c;
        }
      }
#pragma unroll
      for (int v = 0; v < M; ++v) vol[((size_t)e * PD + nd) * M + v] = out[v];
    }
    __syncthreads();
  }
}

// face_integral: d_values [E][P^(D-1) tangential][P_t][m] -> [E][P^D][m]
template <int D, int P>
__global__ void __launch_bounds__(kPieceThreads)
face_integral_kernel(const double* __restrict__ d, int64_t E, int axis, int side, double area,
                     const double* __restrict__ dt_dev, int M, double* __restrict__ out) {
  constexpr int PD = ipow(P, D), PF = PD / P;
  const DegreeTables& T = tab<P>();
  const double dt = *dt_dev;
  const int64_t total = E * PD;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = x / PD;
    const int nd = (int)(x - e * PD);
    int k[3] = {0, 0, 0};
    {
      int r = nd;
      for (int j = D - 1; j >= 0; --j) {
        k[j] = r % P;
        r /= P;
      }
    }
    int tg = 0;
    double wt = 1.0;
    for (int j = 0; j < D; ++j)
      if (j != axis) {
        tg = tg * P + k[j];
        wt *= T.weights[k[j]];
      }
    const double vec = side ? T.right[k[axis]] : T.left[k[axis]];
    const double* src = d + ((size_t)e * PF + tg) * P * M;
    for (int v = 0; v < M; ++v) {
      double db = 0.0;
      for (int t = 0; t < P; ++t) db = fma(T.weights[t], src[t * M + v], db);
      if (D > 1) db = db * wt;
      out[(size_t)x * M + v] = (dt * area) * (vec * db);
    }
  }
}

// extract_traces: q [E][P^D][P_t][m] -> out [D][2][E][P^(D-1)][P_t][m],
// phi(0) / phi(1) contracted along spatial axis j (tangential axes ascending)
template <int D, int P>
__global__ void __launch_bounds__(kPieceThreads)
traces_kernel(const double* __restrict__ q, int64_t E, int m, double* __restrict__ out) {
  constexpr int PD = ipow(P, D), PF = PD / P;
  const DegreeTables& T = tab<P>();
  const int64_t per_dir = E * PF * P;            // (element, tangential node, t)
  const int64_t total = D * per_dir;
  const size_t plane = (size_t)E * PF * P * m;   // one (j, side) output array
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(x / per_dir);
    const int64_t r = x - j * per_dir;
    const int64_t e = r / (PF * P);
    const int tg = (int)((r / P) % PF);
    const int t = (int)(r % P);
    // spatial node of line position l: the tangential digits of tg with l
    // inserted at axis j (row-major, last axis fastest)
    int dig[3] = {0, 0, 0};
    {
      int rem = tg;
      for (int i = D - 1; i >= 0; --i) {
        if (i == j) continue;
        dig[i] = rem % P;
        rem /= P;
      }
    }
    int stride = 1;
    for (int i = D - 1; i > j; --i) stride *= P;
    int base = 0;
    for (int i = 0; i < D; ++i) base = base * P + (i == j ? 0 : dig[i]);
    const double* src = q + ((size_t)e * PD + base) * P * m + (size_t)t * m;
    double* lo = out + (size_t)(2 * j) * plane + ((size_t)r) * m;
    double* hi = lo + plane;
    for (int v = 0; v < m; ++v) {
      double a = 0.0, b = 0.0;
      for (int l = 0; l < P; ++l) {
        const double qv = src[(size_t)l * stride * P * m + v];
        a = fma(T.left[l], qv, a);
        b = fma(T.right[l], qv, b);
      }
      lo[v] = a;
      hi[v] = b;
    }
  }
}

// Space-time rate at every node of q [E][P^D][P_t][m] (Euler):
// conservative L(q) = ((0 - (D/dx_0) F_0) - (D/dx_1) F_1) - .. in the order of
// _rhs_conservative (predictor.py:74-91); primitive primitive_rhs(v, grad v)
// with grad_j = (D/dx_j) v (predictor.py:94-96).  A test hook: every thread
// re-evaluates the fluxes of its P line neighbours per direction.
template <int D, int P>
__global__ void __launch_bounds__(kPieceThreads)
st_rate_kernel(const double* __restrict__ q, int64_t E, double dx0, double dx1, double dx2,
               double gamma, int prim, double* __restrict__ rate) {
  constexpr int M = D + 2, PD = ipow(P, D);
  const DegreeTables& T = tab<P>();
  const double dx[3] = {dx0, dx1, dx2};
  const double gm1 = gamma - 1.0;
  const int64_t total = E * PD * P;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = x / (PD * P);
    const int nd = (int)((x / P) % PD);
    const int t = (int)(x % P);
    int k[3] = {0, 0, 0};
    {
      int rem = nd;
      for (int i = D - 1; i >= 0; --i) {
        k[i] = rem % P;
        rem /= P;
      }
    }
    const double* qe = q + (size_t)e * PD * P * M;
    double out[M], grad[D][M];
#pragma unroll
    for (int v = 0; v < M; ++v) out[v] = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      int stride = 1;
      for (int i = D - 1; i > j; --i) stride *= P;
      const int base = nd - k[j] * stride;
      double acc[M];
#pragma unroll
      for (int v = 0; v < M; ++v) acc[v] = 0.0;
      for (int l = 0; l < P; ++l) {
        const double* ql = qe + ((size_t)(base + l * stride) * P + t) * M;
        double f[M];
        if (prim) {
#pragma unroll
          for (int v = 0; v < M; ++v) f[v] = ql[v];
        } else {
          flux_axis<D>(ql, gm1, j, f);
        }
        const double c = T.diff[k[j] * P + l] / dx[j];   // (diff / spacing)[k][l]
#pragma unroll
        for (int v = 0; v < M; ++v) acc[v] = fma(c, f[v], acc[v]);
      }
#pragma unroll
      for (int v = 0; v < M; ++v) {
        grad[j][v] = acc[v];
        out[v] -= acc[v];
      }
    }
    if (prim) primitive_rhs<D>(qe + ((size_t)nd * P + t) * M, grad, gamma, out);
#pragma unroll
    for (int v = 0; v < M; ++v) rate[(size_t)x * M + v] = out[v];
  }
}

struct AccList {
  const double* p[6];
};

// element_update: u + (vol - acc_0 - acc_1 - ...) / (|cell| w_node)
template <int D, int P>
__global__ void __launch_bounds__(kPieceThreads)
element_update_kernel(const double* __restrict__ u, const double* __restrict__ vol, AccList acc,
                      int nacc, int64_t E, double cv, int M, double* __restrict__ out) {
  constexpr int PD = ipow(P, D);
  const DegreeTables& T = tab<P>();
  const int64_t total = E * PD * M;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int nd = (int)((x / M) % PD);
    double w = T.weights[D == 3 ? nd / (P * P) : (D == 2 ? nd / P : nd)];
    if (D >= 2) w *= T.weights[D == 3 ? (nd / P) % P : nd % P];
    if (D == 3) w *= T.weights[nd % P];
    double tot = vol[x];
    for (int i = 0; i < nacc; ++i) tot -= acc.p[i][x];
    out[x] = u[x] + tot / (cv * w);
  }
}

unsigned grid_for(int64_t work) {
  const int64_t b = (work + kPieceThreads - 1) / kPieceThreads;
  return (unsigned)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

int lerr(std::string* err) {
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

template <int D, int P>
int launch_volume(const adg_grid* g, const double* q, const double* dt, double* vol,
                  cudaStream_t st, std::string* err) {
  const int64_t E = n_elements(g);
  const size_t sm = (size_t)D * ipow(P, D) * (D + 2) * 8;
  static PerDevice attr;
  if (attr.first() && sm > 48 * 1024) {
    if (cudaFuncSetAttribute(volume_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm) != cudaSuccess) {
      *err = "volume tile exceeds shared memory";
      return ADG_ERR_UNSUPPORTED;
    }
  }
  volume_kernel<D, P><<<grid_for(E * kPieceThreads), kPieceThreads, sm, st>>>(
      q, E, g->dx[0], g->dx[1], g->dx[2], g->gamma, dt, vol);
  return lerr(err);
}

template <int D, int P>
int launch_face_integral(const adg_grid* g, int axis, int side, const double* dv,
                         const double* dt, double* out, cudaStream_t st, std::string* err) {
  const int64_t E = n_elements(g);
  // area = prod(spacings) / spacings[axis] as the reference forms it
  double vol = 1.0;
  for (int j = 0; j < g->dim; ++j) vol *= g->dx[j];
  const double area = vol / g->dx[axis];
  face_integral_kernel<D, P><<<grid_for(E * ipow(P, D)), kPieceThreads, 0, st>>>(
      dv, E, axis, side, area, dt, g->nvars, out);
  return lerr(err);
}

template <int D, int P>
int launch_element_update(const adg_grid* g, const double* u, const double* vol,
                          const double* const* accs, int nacc, double* out, cudaStream_t st,
                          std::string* err) {
  const int64_t E = n_elements(g);
  AccList a{};
  for (int i = 0; i < nacc; ++i) a.p[i] = accs[i];
  double cv = 1.0;
  for (int j = 0; j < g->dim; ++j) cv *= g->dx[j];
  element_update_kernel<D, P><<<grid_for(E * ipow(P, D) * g->nvars), kPieceThreads, 0, st>>>(
      u, vol, a, nacc, E, cv, g->nvars, out);
  return lerr(err);
}

template <int D, int P>
int launch_traces(const adg_grid* g, const double* q, double* out, cudaStream_t st,
                  std::string* err) {
  const int64_t E = n_elements(g);
  traces_kernel<D, P><<<grid_for(E * D * ipow(P, D)), kPieceThreads, 0, st>>>(q, E, g->nvars,
                                                                             out);
  return lerr(err);
}

template <int D, int P>
int launch_st_rate(const adg_grid* g, const double* q, double* rate, cudaStream_t st,
                   std::string* err) {
  const int64_t E = n_elements(g);
  st_rate_kernel<D, P><<<grid_for(E * ipow(P, D + 1)), kPieceThreads, 0, st>>>(
      q, E, g->dx[0], g->dx[1], g->dx[2], g->gamma, g->mode == ADG_MODE_PRIMITIVE ? 1 : 0, rate);
  return lerr(err);
}

}  // namespace

#define ADG_PIECE_SWITCH(FN, ...)                          \
  do {                                                     \
    const int P = g->degree + 1;                           \
    switch (g->dim * 16 + P) {                             \
      case 17: return FN<1, 1>(__VA_ARGS__);               \
      case 18: return FN<1, 2>(__VA_ARGS__);               \
      case 19: return FN<1, 3>(__VA_ARGS__);               \
      case 20: return FN<1, 4>(__VA_ARGS__);               \
      case 21: return FN<1, 5>(__VA_ARGS__);               \
      case 22: return FN<1, 6>(__VA_ARGS__);               \
      case 23: return FN<1, 7>(__VA_ARGS__);               \
      case 24: return FN<1, 8>(__VA_ARGS__);               \
      case 25: return FN<1, 9>(__VA_ARGS__);               \
      case 26: return FN<1, 10>(__VA_ARGS__);              \
      case 33: return FN<2, 1>(__VA_ARGS__);               \
      case 34: return FN<2, 2>(__VA_ARGS__);               \
      case 35: return FN<2, 3>(__VA_ARGS__);               \
      case 36: return FN<2, 4>(__VA_ARGS__);               \
      case 37: return FN<2, 5>(__VA_ARGS__);               \
      case 38: return FN<2, 6>(__VA_ARGS__);               \
      case 39: return FN<2, 7>(__VA_ARGS__);               \
      case 40: return FN<2, 8>(__VA_ARGS__);               \
      case 41: return FN<2, 9>(__VA_ARGS__);               \
      case 42: return FN<2, 10>(__VA_ARGS__);              \
      case 49: return FN<3, 1>(__VA_ARGS__);               \
      case 50: return FN<3, 2>(__VA_ARGS__);               \
      case 51: return FN<3, 3>(__VA_ARGS__);               \
      case 52: return FN<3, 4>(__VA_ARGS__);               \
      case 53: return FN<3, 5>(__VA_ARGS__);               \
      case 54: return FN<3, 6>(__VA_ARGS__);               \
      case 55: return FN<3, 7>(__VA_ARGS__);               \
      case 56: return FN<3, 8>(__VA_ARGS__);               \
      case 57: return FN<3, 9>(__VA_ARGS__);               \
      case 58: return FN<3, 10>(__VA_ARGS__);              \
    }                                                      \
    *err = "unsupported dim/degree";                       \
    return ADG_ERR_UNSUPPORTED;                            \
  } while (0)

int face_points(const adg_grid* g, int axis, int64_t n, const double* qm, const double* qp,
                double* dlow, double* dhigh, cudaStream_t st, std::string* err) {
  if (n <= 0) return ADG_OK;
  const unsigned grid = grid_for(n);
  if (g->dim == 1) face_points_kernel<1><<<grid, kPieceThreads, 0, st>>>(qm, qp, n, axis, g->gamma, dlow, dhigh);
  if (g->dim == 2) face_points_kernel<2><<<grid, kPieceThreads, 0, st>>>(qm, qp, n, axis, g->gamma, dlow, dhigh);
  if (g->dim == 3) face_points_kernel<3><<<grid, kPieceThreads, 0, st>>>(qm, qp, n, axis, g->gamma, dlow, dhigh);
  return lerr(err);
}

int riemann_points(const adg_grid* g, int64_t n, const double* normal, int mode,
                   const double* qm, const double* qp, double* out_a, double* out_b,
                   cudaStream_t st, std::string* err) {
  if (n <= 0) return ADG_OK;
  const unsigned grid = grid_for(n);
  const double* a = g->velocity;
#define ADG_RIEMANN(SYS, D)                                                                 \
  riemann_points_kernel<SYS, D><<<grid, kPieceThreads, 0, st>>>(                            \
      qm, qp, n, normal[0], normal[1], normal[2], g->gamma, a[0], a[1], a[2], mode, out_a, \
      out_b)
  const int sys = g->system == ADG_SYS_ADVECTION ? 1 : 0;
  if (sys == 0 && g->dim == 1) ADG_RIEMANN(0, 1);
  if (sys == 0 && g->dim == 2) ADG_RIEMANN(0, 2);
  if (sys == 0 && g->dim == 3) ADG_RIEMANN(0, 3);
  if (sys == 1 && g->dim == 1) ADG_RIEMANN(1, 1);
  if (sys == 1 && g->dim == 2) ADG_RIEMANN(1, 2);
  if (sys == 1 && g->dim == 3) ADG_RIEMANN(1, 3);
#undef ADG_RIEMANN
  return lerr(err);
}


int lim_minmod(const double* a, const double* b, int64_t n, double* out, cudaStream_t st,
               std::string* err) {
  if (n <= 0) return ADG_OK;
  minmod_kernel<<<grid_for(n), kPieceThreads, 0, st>>>(a, b, n, out);
  return lerr(err);
}

int lim_relaxed_bounds(int dim, int m, const int64_t* cells, int nsub, const double* padded_sub,
                       double delta0, double eps, double* cmin_pad, double* cmax_pad, double* lo,
                       double* hi, cudaStream_t st, std::string* err) {
  int64_t npad = 1, ncore = 1;
  for (int j = 0; j < dim; ++j) {
    npad *= cells[j] + 2;
    ncore *= cells[j];
  }
  if (ncore <= 0) return ADG_OK;
  cell_extrema_kernel<<<grid_for(npad * m), kPieceThreads, 0, st>>>(padded_sub, npad, nsub, m,
                                                                    cmin_pad, cmax_pad);
  relaxed_bounds_kernel<<<grid_for(ncore * m), kPieceThreads, 0, st>>>(
      cmin_pad, cmax_pad, dim, cells[0], dim >= 2 ? cells[1] : 1, dim == 3 ? cells[2] : 1, m,
      delta0, eps, lo, hi);
  return lerr(err);
}

int lim_detect_cells(const adg_grid* g, const double* cand, const double* sub, const double* lo,
                     const double* hi, uint8_t* out, cudaStream_t st, std::string* err) {
  const int64_t E = n_elements(g);
  if (E <= 0) return ADG_OK;
  const int P = g->degree + 1, S = 2 * g->degree + 1;
  int pd = 1, sd = 1;
  for (int j = 0; j < g->dim; ++j) {
    pd *= P;
    sd *= S;
  }
  const unsigned grid = grid_for(E);
  const double gm1 = g->gamma - 1.0;
  const int m = g->nvars;
  if (g->system == ADG_SYS_EULER) {
    if (g->dim == 1) detect_cells_kernel<0, 1><<<grid, kPieceThreads, 0, st>>>(cand, sub, lo, hi, E, pd, sd, m, gm1, out);
    if (g->dim == 2) detect_cells_kernel<0, 2><<<grid, kPieceThreads, 0, st>>>(cand, sub, lo, hi, E, pd, sd, m, gm1, out);
    if (g->dim == 3) detect_cells_kernel<0, 3><<<grid, kPieceThreads, 0, st>>>(cand, sub, lo, hi, E, pd, sd, m, gm1, out);
  } else {
    detect_cells_kernel<1, 1><<<grid, kPieceThreads, 0, st>>>(cand, sub, lo, hi, E, pd, sd, m, gm1, out);
  }
  return lerr(err);
}

int lim_gather_windows(int dim, int m, const int64_t* dims, const double* padded,
                       const int64_t* starts, int64_t nwin, int size, double* out,
                       cudaStream_t st, std::string* err) {
  int64_t per = m;
  for (int j = 0; j < dim; ++j) per *= size;
  if (nwin * per <= 0) return ADG_OK;
  gather_windows_kernel<<<grid_for(nwin * per), kPieceThreads, 0, st>>>(
      padded, dim, dims[0], dim >= 2 ? dims[1] : 1, dim == 3 ? dims[2] : 1, m, starts, nwin, size,
      out);
  return lerr(err);
}

int volume_integral(const adg_grid* g, const double* q, const double* dt_dev, double* vol,
                    cudaStream_t st, std::string* err) {
  ADG_PIECE_SWITCH(launch_volume, g, q, dt_dev, vol, st, err);
}

int face_integral(const adg_grid* g, int axis, int side, const double* d_values,
                  const double* dt_dev, double* out, cudaStream_t st, std::string* err) {
  ADG_PIECE_SWITCH(launch_face_integral, g, axis, side, d_values, dt_dev, out, st, err);
}

int extract_traces(const adg_grid* g, const double* q, double* out, cudaStream_t st,
                   std::string* err) {
  ADG_PIECE_SWITCH(launch_traces, g, q, out, st, err);
}

int spacetime_rate(const adg_grid* g, const double* q, double* rate, cudaStream_t st,
                   std::string* err) {
  ADG_PIECE_SWITCH(launch_st_rate, g, q, rate, st, err);
}

int element_update(const adg_grid* g, const double* u, const double* vol,
                   const double* const* accs, int nacc, double* out, cudaStream_t st,
                   std::string* err) {
  ADG_PIECE_SWITCH(launch_element_update, g, u, vol, accs, nacc, out, st, err);
}

}  // namespace adg
