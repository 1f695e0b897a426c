// adg_pieces.cu -- the reference's corrector module functions as standalone
// device calls (sm_100a), for callers that use the module API directly
// instead of Simulation (SURVEY.md §8(b) "module functions"):
//   face_fluxes     (corrector.py:100-129)  pointwise Rusanov pair
//   volume_integral (corrector.py:141-177)  from a given space-time q
//   face_integral   (corrector.py:180-196)  one face's accumulator
//   element_update  (corrector.py:199-205)  u + (vol - sum faces) / mass
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
                     const double* __restrict__ dt_dev, double* __restrict__ out) {
  constexpr int M = D + 2, PD = ipow(P, D), PF = PD / P;
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
#pragma unroll
    for (int v = 0; v < M; ++v) {
      double db = 0.0;
      for (int t = 0; t < P; ++t) db = fma(T.weights[t], src[t * M + v], db);
      if (D > 1) db = db * wt;
      out[(size_t)x * M + v] = (dt * area) * (vec * db);
    }
  }
}

struct AccList {
  const double* p[6];
};

// element_update: u + (vol - acc_0 - acc_1 - ...) / (|cell| w_node)
template <int D, int P>
__global__ void __launch_bounds__(kPieceThreads)
element_update_kernel(const double* __restrict__ u, const double* __restrict__ vol, AccList acc,
                      int nacc, int64_t E, double cv, double* __restrict__ out) {
  constexpr int M = D + 2, PD = ipow(P, D);
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
      dv, E, axis, side, area, dt, out);
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
  element_update_kernel<D, P><<<grid_for(E * ipow(P, D) * (D + 2)), kPieceThreads, 0, st>>>(
      u, vol, a, nacc, E, cv, out);
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

int volume_integral(const adg_grid* g, const double* q, const double* dt_dev, double* vol,
                    cudaStream_t st, std::string* err) {
  ADG_PIECE_SWITCH(launch_volume, g, q, dt_dev, vol, st, err);
}

int face_integral(const adg_grid* g, int axis, int side, const double* d_values,
                  const double* dt_dev, double* out, cudaStream_t st, std::string* err) {
  ADG_PIECE_SWITCH(launch_face_integral, g, axis, side, d_values, dt_dev, out, st, err);
}

int element_update(const adg_grid* g, const double* u, const double* vol,
                   const double* const* accs, int nacc, double* out, cudaStream_t st,
                   std::string* err) {
  ADG_PIECE_SWITCH(launch_element_update, g, u, vol, accs, nacc, out, st, err);
}

}  // namespace adg
