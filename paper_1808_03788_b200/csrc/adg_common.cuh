// adg_common.cuh -- shared device code of libaderdg_b200.so (sm_100a).
//
// Per-degree constant tables (basis.py:166-202, predictor.py:21-47) live in
// __constant__ memory for every degree 0..9 at once, so kernels templated on
// P = N+1 index them at compile time (uniform access -> constant cache).
// Euler pointwise physics follows systems.py:112-234 operation by operation.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/aderdg_b200.h"

namespace adg {

constexpr int kMaxP = 10;
constexpr int kMaxS = 2 * kMaxP - 1;

struct DegreeTables {
  double nodes[kMaxP];
  double weights[kMaxP];
  double diff[kMaxP * kMaxP];     // diff[k*P + l] = ell_l'(xi_k)
  double left[kMaxP];
  double right[kMaxP];
  double gw[kMaxP * kMaxP];       // K1^-1 diag(w)
  double g0[kMaxP];               // K1^-1 phi(0)
  double k1_opnorm;
  double sub_project[kMaxS * kMaxP];  // [S][P]
  double sub_recover[kMaxP * kMaxS];  // [P][S]
  double stiff[kMaxP * kMaxP];    // stiff[k*P+l] = diff[l*P+k] * w[l]  (corrector.py:168)
  int loaded;
};

extern __constant__ DegreeTables c_tab[kMaxP];
extern DegreeTables h_tab[kMaxP];   // host copy (adg_set_tables)

template <int P> __device__ __forceinline__ const DegreeTables& tab() { return c_tab[P - 1]; }

__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// ---------------------------------------------------------------- Euler
// 1/x from the hardware approximation refined by two Newton steps (error
// below one ulp of the IEEE quotient; the reference's 1.0 / rho is replaced
// at the 1e-16 level, far inside the 1e-10 parity bar).  Saves the
// slow-path-guarded IEEE division on every flux evaluation.
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// systems.py:128-133 pressure; identical operation order.
template <int D>
__device__ __forceinline__ double pressure(const double* q, double gm1) {
  double kin = q[1] * q[1];
#pragma unroll
  for (int j = 1; j < D; ++j) kin = kin + q[1 + j] * q[1 + j];
  return gm1 * (q[D + 1] - 0.5 * kin / q[0]);
}

// systems.py:140-156: F[j][v].  One IEEE division (1/rho) as in the reference.
template <int D>
__device__ __forceinline__ void flux_all(const double* q, double gm1, double f[D][D + 2]) {
  const double r = rcp_nr(q[0]);
  double kin = q[1] * q[1];
#pragma unroll
  for (int j = 1; j < D; ++j) kin = kin + q[1 + j] * q[1 + j];
  const double p = gm1 * (q[D + 1] - 0.5 * kin * r);
  const double ep = q[D + 1] + p;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double vj = q[1 + j] * r;
    f[j][0] = q[1 + j];
#pragma unroll
    for (int i = 0; i < D; ++i) f[j][1 + i] = q[1 + i] * vj;
    f[j][1 + j] += p;
    f[j][D + 1] = ep * vj;
  }
}

// Flux along a single axis a (same arithmetic as flux_all's row a).
template <int D>
__device__ __forceinline__ void flux_axis(const double* q, double gm1, int a, double f[D + 2]) {
  const double r = rcp_nr(q[0]);
  double kin = q[1] * q[1];
#pragma unroll
  for (int j = 1; j < D; ++j) kin = kin + q[1 + j] * q[1 + j];
  const double p = gm1 * (q[D + 1] - 0.5 * kin * r);
  const double ep = q[D + 1] + p;
  const double va = q[1 + a] * r;
  f[0] = q[1 + a];
#pragma unroll
  for (int i = 0; i < D; ++i) f[1 + i] = q[1 + i] * va;
  f[1 + a] += p;
  f[D + 1] = ep * va;
}

// flux_axis with a runtime axis (one instruction stream for every axis):
// the normal momentum is selected, and the pressure enters its row through
// the fma addend (zero elsewhere: fma(q, v, 0) is the rounded product)
template <int D>
__device__ __forceinline__ void flux_axis_dyn(const double* q, double gm1, int a,
                                              double f[D + 2]) {
  const double r = rcp_nr(q[0]);
  double kin = q[1] * q[1];
#pragma unroll
  for (int j = 1; j < D; ++j) kin = kin + q[1 + j] * q[1 + j];
  const double p = gm1 * (q[D + 1] - 0.5 * kin * r);
  const double ep = q[D + 1] + p;
  double ma = q[1];
#pragma unroll
  for (int j = 1; j < D; ++j) ma = a == j ? q[1 + j] : ma;
  const double va = ma * r;
  f[0] = ma;
#pragma unroll
  for (int i = 0; i < D; ++i) f[1 + i] = fma(q[1 + i], va, a == i ? p : 0.0);
  f[D + 1] = ep * va;
}

// systems.py:173-178 with normal e_a: |u_n / rho| + sqrt(gamma p / rho),
// u_n accumulated as 0 + sum_j q_j n_j exactly like the reference.
template <int D>
__device__ __forceinline__ double max_abs_eig(const double* q, double gamma, double gm1, int a) {
  double un = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) un = un + q[1 + j] * (j == a ? 1.0 : 0.0);
  const double p = pressure<D>(q, gm1);
  return fabs(un / q[0]) + sqrt(gamma * p / q[0]);
}

// Flux along axis a AND the max |eigenvalue| of the same state, sharing one
// reciprocal of rho and one pressure (face kernel: corrector.py:58-62 +
// systems.py:140-178).  Quotients become products with the Newton-refined
// reciprocal (<= 1 ulp), so lam may differ from the reference's in the last
// bit; it only scales the Rusanov dissipation.
template <int D>
__device__ __forceinline__ double flux_eig_axis(const double* q, double gamma, double gm1, int a,
                                                double f[D + 2]) {
  const double r = rcp_nr(q[0]);
  double kin = q[1] * q[1];
#pragma unroll
  for (int j = 1; j < D; ++j) kin = kin + q[1 + j] * q[1 + j];
  const double p = gm1 * (q[D + 1] - 0.5 * kin * r);
  const double ep = q[D + 1] + p;
  const double va = q[1 + a] * r;
  f[0] = q[1 + a];
#pragma unroll
  for (int i = 0; i < D; ++i) f[1 + i] = q[1 + i] * va;
  f[1 + a] += p;
  f[D + 1] = ep * va;
  return fabs(va) + sqrt(gamma * p * r);
}

// systems.py:180-198 conservative <-> primitive (rho, v_1..d, p)
template <int D>
__device__ __forceinline__ void cons_to_prim(const double* q, double gm1, double* v) {
  v[0] = q[0];
#pragma unroll
  for (int j = 0; j < D; ++j) v[1 + j] = q[1 + j] / q[0];
  v[D + 1] = pressure<D>(q, gm1);
}
template <int D>
__device__ __forceinline__ void prim_to_cons(const double* v, double gm1, double* q) {
  const double rho = v[0];
  double kin = v[1] * v[1];
#pragma unroll
  for (int j = 1; j < D; ++j) kin = kin + v[1 + j] * v[1 + j];
  q[0] = rho;
#pragma unroll
  for (int j = 0; j < D; ++j) q[1 + j] = rho * v[1 + j];
  q[D + 1] = v[D + 1] / gm1 + 0.5 * rho * kin;
}

// systems.py:200-223: quasi-linear primitive time derivative; g[j][w] is
// the j-derivative of primitive quantity w
template <int D>
__device__ __forceinline__ void primitive_rhs(const double* v, const double g[D][D + 2],
                                              double gamma, double* out) {
  const double rho = v[0], p = v[D + 1];
  double div = g[0][1];
#pragma unroll
  for (int j = 1; j < D; ++j) div = div + g[j][1 + j];
  double arho = v[1] * g[0][0];
  double ap = v[1] * g[0][D + 1];
#pragma unroll
  for (int j = 1; j < D; ++j) {
    arho = arho + v[1 + j] * g[j][0];
    ap = ap + v[1 + j] * g[j][D + 1];
  }
  out[0] = -(arho + rho * div);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double av = v[1] * g[0][1 + i];
#pragma unroll
    for (int j = 1; j < D; ++j) av = av + v[1 + j] * g[j][1 + i];
    out[1 + i] = -(av + g[i][D + 1] / rho);
  }
  out[D + 1] = -(ap + gamma * p * div);
}

// systems.py:225-229: all finite, rho > 0, p > 0.
template <int D>
__device__ __forceinline__ bool admissible(const double* q, double gm1) {
  bool fin = true;
#pragma unroll
  for (int v = 0; v < D + 2; ++v) fin = fin && isfinite(q[v]);
  const double p = pressure<D>(q, gm1);
  return fin && (q[0] > 0.0) && (p > 0.0);
}

// systems.py:225-229 with the sign of p read from a Newton-refined
// reciprocal of rho: within 1e-12 of cancellation the reference's IEEE
// division decides, so the verdict equals admissible<D>'s exactly
template <int D>
__device__ __forceinline__ bool admissible_fast(const double* q, double gm1) {
  bool fin = true;
#pragma unroll
  for (int v = 0; v < D + 2; ++v) fin = fin && isfinite(q[v]);
  if (!fin || !(q[0] > 0.0)) return false;
  const double r = rcp_nr(q[0]);
  double kin = q[1] * q[1];
#pragma unroll
  for (int j = 1; j < D; ++j) kin = kin + q[1 + j] * q[1 + j];
  const double x = 0.5 * kin * r;
  const double dd = q[D + 1] - x;
  if (fabs(dd) > 1e-12 * (fabs(q[D + 1]) + fabs(x))) return dd > 0.0;
  return pressure<D>(q, gm1) > 0.0;
}

// flux_all and admissible of one state sharing the reciprocal of rho: the
// sign of p = gm1 (E - 0.5 kin / rho) is read from the reciprocal-based
// E - 0.5 kin r, which is within a few ulp of the reference's quotient; only
// within 1e-12 of cancellation is the reference's IEEE division evaluated,
// so the verdict is exactly systems.py:225-229's.
template <int D>
__device__ __forceinline__ bool flux_all_adm(const double* q, double gm1, double f[D][D + 2]) {
  const double r = rcp_nr(q[0]);
  double kin = q[1] * q[1];
#pragma unroll
  for (int j = 1; j < D; ++j) kin = kin + q[1 + j] * q[1 + j];
  const double x = 0.5 * kin * r;
  const double dd = q[D + 1] - x;
  const double p = gm1 * dd;
  const double ep = q[D + 1] + p;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double vj = q[1 + j] * r;
    f[j][0] = q[1 + j];
#pragma unroll
    for (int i = 0; i < D; ++i) f[j][1 + i] = q[1 + i] * vj;
    f[j][1 + j] += p;
    f[j][D + 1] = ep * vj;
  }
  bool fin = true;
#pragma unroll
  for (int v = 0; v < D + 2; ++v) fin = fin && isfinite(q[v]);
  bool ppos;
  if (fabs(dd) > 1e-12 * (fabs(q[D + 1]) + fabs(x))) ppos = dd > 0.0;
  else ppos = pressure<D>(q, gm1) > 0.0;
  return fin && (q[0] > 0.0) && ppos;
}

// max of two wave speeds with numpy's np.maximum semantics: a NaN in either
// operand propagates (fmax would return the other one).  A face state with
// negative pressure has a NaN sound speed; the reference's Rusanov term and
// hence the candidate become NaN there and the limiter takes the cell
// (corrector.py:58-62, limiter.py:76-86).
__device__ __forceinline__ double nan_max(double a, double b) {
  return (a >= b || a != a) ? a : b;
}

// Rusanov one-sided terms (corrector.py:100-129) for a subcell face
template <int D>
__device__ __forceinline__ void rusanov_pair(const double* qm, const double* qp, int a,
                                             double gamma, double gm1, double* dlow,
                                             double* dhigh) {
  constexpr int M = D + 2;
  const double s = nan_max(max_abs_eig<D>(qm, gamma, gm1, a), max_abs_eig<D>(qp, gamma, gm1, a));
  double fm[M], fp[M];
  flux_axis<D>(qm, gm1, a, fm);
  flux_axis<D>(qp, gm1, a, fp);
  const double hs = 0.5 * s;
#pragma unroll
  for (int v = 0; v < M; ++v) {
    const double central = 0.5 * (fm[v] + fp[v]);
    const double diss = hs * (qp[v] - qm[v]);
    dlow[v] = (central + 0.0) - diss;
    dhigh[v] = (-central + 0.0) + diss;
  }
}

__device__ __forceinline__ double minmod(double a, double b) {
  return (a * b > 0.0) ? (fabs(a) <= fabs(b) ? a : b) : 0.0;
}

__device__ __forceinline__ void atomic_max_pos(uint64_t* addr, double v) {
  // v >= 0 and finite: IEEE bit patterns order like unsigned integers
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

// ---------------------------------------------------------------- TMA bulk
// 1-D bulk copies between global and shared memory (cp.async.bulk, SASS
// UBLKCP) completing on an mbarrier; sizes and addresses 16-byte aligned.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// per-thread asynchronous 8-byte global -> shared copies (SASS LDGSTS):
// prefetch of the next element's state while the current one computes
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
// all but the most recently committed group have landed
__device__ __forceinline__ void cp_async_wait_1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Host-side launch helpers ------------------------------------------------
struct LaunchCtx {
  cudaStream_t stream;
  int num_sms;
};

}  // namespace adg
