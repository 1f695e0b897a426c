// adg_predictor_phased.cu -- the ADER-DG predictor for the large 3-D
// space-time tiles (P = N+1 = 8..10: 160-391 KB per element, more than one
// SM's shared memory) as a sequence of phase kernels over a batch of
// elements, the space-time iterate and its rates in HBM.
//
// Same algorithm and outputs as predict_kernel (adg_predictor.cu): startup
// guess (predictor.py:99-126), Picard sweeps with per-element freezing
// (predictor.py:135-191), admissibility (:188-189), face traces (:218-230)
// and the volume integral (corrector.py:141-177).
//
// Why phases.  A fused per-element kernel at these degrees holds one 30-40 KB
// time slice and 45-50 line accumulators per thread: one CTA of 9 warps per SM,
// every slice a serial load -> contract -> store chain (measured: 75 % of the
// cycles without an eligible warp, FP64 pipe at 17 %).  B200 has 6.5 TB/s of
// HBM for 37 TFLOP/s of FP64, so the tile can afford to travel: the Picard
// rate L(q_t) = -sum_dir D_dir F_dir(q_t) only couples the nodes of ONE time
// slice and the time operator only the time levels of ONE node, so
//   startup  one CTA per element: k1 = L(u), k2 = L(u + dt k1), q_t at every t;
//   rates    one CTA per (element, time slice): slice -> shared memory, the
//            P^2 line owners contract z, y, x flux lines (one shared partial
//            buffer, accumulated in place), rate slice -> HBM;
//   time     one CTA per element, streaming: q_new = dt gw rate + g0 u,
//            residual, convergence flag, q <- q_new;
//   final    one CTA per element: traces, admissibility, flux sums, volume.
// Slices are independent tasks, so every SM holds several CTAs in different
// phases of their slices, and each pass streams at HBM speed.  Frozen
// elements are skipped by every later rates / time launch; a device counter
// of active elements turns the remaining launches of the host's max_iter
// loop into immediate exits (no host synchronisation, graph-capturable).
#include <algorithm>
#include <cstdlib>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

// l loop of the line contractions: fully unrolled by default (D/dx entries
// become constant-bank operands; measured 34.5 vs 35.1 ms at N = 8, 58.6 vs
// 63.2 ms at N = 9 against the rolled loop)
#ifndef ADG_PH_LUNROLL
#define ADG_PH_LUNROLL 16
#endif
// 1 / rho and the pressure of every node of the slice computed once into
// shared memory (instead of once per direction by the line owners)
// (measured 2-7 % SLOWER at N = 7..9: the kernel is latency-bound, not
// FP64-issue-bound, and the extra shared traffic costs more than the saved
// flux arithmetic; kept for A/B builds)
#ifndef ADG_PH_RP
#define ADG_PH_RP 0
#endif
// output halves per line: with NH = 2 two warp groups own the same lines and
// each accumulates half of the P outputs (half the accumulator registers,
// twice the warps per CTA; the line's fluxes are formed by both)
#ifndef ADG_PH_NH
#define ADG_PH_NH 1
#endif
// (node, quantity) items per thread in flight in the time kernel
#ifndef ADG_PH_TNB
#define ADG_PH_TNB 1
#endif
// CTAs per SM the time kernel is compiled for (register cap 65536 / (256 n))
#ifndef ADG_PH_FMINB
#define ADG_PH_FMINB 2   // flux-sums kernel: 128 registers hold the pipelined loads (3: spills, +0.8 ms at N = 8)
#endif
#ifndef ADG_PH_TMINB
#define ADG_PH_TMINB (ADG_PH_TNB == 1 ? 3 : 2)
#endif


template <int P>
struct PhCfg {
  static constexpr int M = 5;
  static constexpr int PP = P * P;
  static constexpr int PD = P * P * P;
  // padded slice layouts (tools/slice_bankcheck.py): Q node-major
  // [i][j][k][v] strides (SI, SJ, M); B x-line-major [j][k][i][v] strides
  // (TJ, TK, M)
  static constexpr int SJ = P * M + (P == 8 ? 1 : (P == 10 ? 3 : 0));
  static constexpr int SI = P * SJ;
  static constexpr int TK = P * M + (P == 8 ? 2 : (P == 10 ? 1 : 0));
  static constexpr int TJ = P * TK + (P == 8 ? 1 : 0);
  static constexpr int QSZ = P * SI;
  static constexpr int BSZ = P * TJ;
  static constexpr int QSZP = QSZ + (QSZ & 1);
  // (the partial buffer also stages a stored slice in the first sweep)
  static constexpr int BSZP = (BSZ > QSZ ? BSZ : QSZ) + ((BSZ > QSZ ? BSZ : QSZ) & 1);
  static constexpr int RP = ((PP + 31) / 32) * 32;   // line owners, whole warps
  static constexpr int NH = ADG_PH_NH;
  static constexpr int H = (P + NH - 1) / NH;        // outputs per thread
  static constexpr int NT_A = NH * RP;               // threads of the line kernels
  static constexpr int NW = NT_A / 32;
  static constexpr int CSTP = (2 * P + 1) / 2 * 2;
  static constexpr size_t SLICE = (size_t)PD * M;    // doubles per time slice
  static constexpr size_t TILE = (size_t)P * SLICE;  // doubles per space-time tile
  // the iterate is stored slice by slice in the PADDED shared-memory layout
  // (QSZP doubles, even: 16-byte aligned), so a slice lands in shared memory
  // with one bulk copy (cp.async.bulk, TMA) instead of P^3 m 8-byte copies
  static constexpr size_t TILEQ = (size_t)P * QSZP;
  static constexpr bool DENSE = (SJ == P * M) && (SI == P * SJ);
  static constexpr int TB = PD * M + ((PD * M) & 1); // trace block (face kernel layout)
  // rates / startup: one slice + one partial buffer
  static constexpr int XSZ = ADG_PH_RP ? 2 * PD : 0;   // (1 / rho, p) per node
  static constexpr size_t SMEM_A = ((size_t)QSZP + BSZP + XSZ) * 8;
  // register cap of the line kernels: 168 per thread (a warp's registers
  // come from its scheduler's 16 K: more would cost the third CTA per SM)
  static constexpr int MINB_A = NH == 1 ? 384 / RP : (640 / NT_A > 0 ? 640 / NT_A : 1);
  // traces: one slice, three line-owner groups side by side
  static constexpr int NT_F = 3 * RP;
  static constexpr int TRS = 6 * PP * M;             // staged traces of one slice
  static constexpr size_t SMEM_TR = ((size_t)QSZP + TRS) * 8;
  static constexpr int MINB_TR = NT_F > 288 ? 3 : 4;
  // vol: slice + y partials + z partials
  static constexpr size_t SMEM_V = ((size_t)QSZP + 2 * BSZP) * 8;
  static constexpr int NT_T = 256;                   // time kernel

};

struct PhArgs {
  const double* u;      // batch's first element
  const double* dt;
  double* q_out;        // batch's first element, or null
  double* vol;
  double* traces;       // batch's first element inside face plane 0
  uint8_t* pred_bad;
  int32_t* sweeps;
  double* qg;           // [n][P][node][v] iterate
  double* rg;           // [n][P][node][v] rates; after the sweeps slices 0..2 = Fbar_x/y/z
  double* kg;           // [n][3] stored (padded) slices: u, k1, k2 - k1
  int32_t* state;       // [4][n]: frozen, converged, sweeps executed, inadmissible
  int32_t* n_active;
  int64_t n_elem;       // elements in the batch
  int64_t tr_elems;     // elements per face plane of the trace array
  double dx[3];
  double gamma;
  double tol;
  int max_iter;
  int min_iter;
  int it;               // sweep index (rates / time launches)
  double dd[3 * kMaxP * kMaxP];   // D / dx_dir, [dir][P][P]
};

// one line's P states (src + l * stride) -> flux along DIR -> D/dx_DIR
// contraction, l-outer: every line state is loaded, turned into its flux and
// folded into all P outputs (same per-output fma order as a row-by-row
// mat-vec)
template <int P, int DIR, int HF>
__device__ __forceinline__ void ph_line_h(const double* src0, int stride, const double* x0,
                                          int xstride, double gm1, const double* dd,
                                          double (&acc)[PhCfg<P>::H][5]) {
  constexpr int M = 5, H = PhCfg<P>::H, IB = HF * H;
#pragma unroll
  for (int i = 0; i < H; ++i)
#pragma unroll
    for (int v = 0; v < M; ++v) acc[i][v] = 0.0;
  constexpr int LU = ADG_PH_LUNROLL;
#pragma unroll LU
  for (int l = 0; l < P; ++l) {
    double q[M], f[M];
    const double* src = src0 + l * stride;
#pragma unroll
    for (int v = 0; v < M; ++v) q[v] = src[v];
    if constexpr (ADG_PH_RP) {
      // flux_axis with the node's 1 / rho and p from the slice pre-pass (the
      // same values flux_axis would form)
      const double2 rp = *reinterpret_cast<const double2*>(x0 + l * xstride);
      const double va = q[1 + DIR] * rp.x;
      const double ep = q[4] + rp.y;
      f[0] = q[1 + DIR];
#pragma unroll
      for (int i = 0; i < 3; ++i) f[1 + i] = q[1 + i] * va;
      f[1 + DIR] += rp.y;
      f[4] = ep * va;
    } else {
      flux_axis<3>(q, gm1, DIR, f);
    }
#pragma unroll
    for (int i = 0; i < H; ++i) {
      if (IB + i < P) {
        const double d = dd[DIR * P * P + (IB + i) * P + l];
#pragma unroll
        for (int v = 0; v < M; ++v) acc[i][v] = fma(d, f[v], acc[i][v]);
      }
    }
  }
}
template <int P, int DIR>
__device__ __forceinline__ void ph_line(const double* src0, int stride, const double* x0,
                                        int xstride, double gm1, const double* dd, int half,
                                        double (&acc)[PhCfg<P>::H][5]) {
  if (PhCfg<P>::NH == 1 || half == 0)
    ph_line_h<P, DIR, 0>(src0, stride, x0, xstride, gm1, dd, acc);
  else
    ph_line_h<P, DIR, PhCfg<P>::NH - 1>(src0, stride, x0, xstride, gm1, dd, acc);
}

// 1 / rho and p of every node of the padded slice Q -> X[node] (node-major,
// unpadded), exactly as flux_axis forms them
template <int P, int NT>
__device__ __forceinline__ void ph_prepass(const double* Q, double* X, double gm1, int tid) {
  using C = PhCfg<P>;
  if constexpr (ADG_PH_RP) {
    for (int n = tid; n < C::PD; n += NT) {
      const int i = n / C::PP, j = (n / P) % P, k = n % P;
      const double* q = Q + i * C::SI + j * C::SJ + k * C::M;
      const double r = rcp_nr(q[0]);
      double kin = q[1] * q[1];
      kin = kin + q[2] * q[2];
      kin = kin + q[3] * q[3];
      const double pr = gm1 * (q[4] - 0.5 * kin * r);
      *reinterpret_cast<double2*>(X + 2 * n) = make_double2(r, pr);
    }
    __syncthreads();
  }
}

// the line-owner indices of thread rr (< P^2) in the three roles
template <int P>
struct PhRoles {
  int a0, b0;
  __device__ __forceinline__ explicit PhRoles(int rr) : a0(rr / P), b0(rr - (rr / P) * P) {}
  using C = PhCfg<P>;
  // first node of the owned line in the padded slice, and the line's stride
  __device__ __forceinline__ int qbase(int role) const {
    return role == 0 ? a0 * C::SJ + b0 * C::M
                     : (role == 1 ? a0 * C::SI + b0 * C::M : a0 * C::SI + b0 * C::SJ);
  }
  __device__ __forceinline__ int qstride(int role) const {
    return role == 0 ? C::SI : (role == 1 ? C::SJ : C::M);
  }
  // unpadded node index of the line's first node and the node stride
  __device__ __forceinline__ int nbase(int role) const {
    return role == 0 ? a0 * P + b0 : (role == 1 ? a0 * C::PP + b0 : a0 * C::PP + b0 * P);
  }
  __device__ __forceinline__ int nstride(int role) const {
    return role == 0 ? C::PP : (role == 1 ? P : 1);
  }
  // where the y (role 1) / z (role 2) owner's output i lands in the
  // x-line-major partial buffer: pbase + i * pstride
  __device__ __forceinline__ int pbase(int role) const {
    return role == 1 ? b0 * C::TK + a0 * C::M : b0 * C::TJ + a0 * C::M;
  }
  __device__ __forceinline__ int pstride(int role) const { return role == 1 ? C::TJ : C::TK; }
  __device__ __forceinline__ int xrow() const { return a0 * C::TJ + b0 * C::TK; }
};

// offset of the x-th double of a [node][v] slice in the padded slice layout
template <int P>
__device__ __forceinline__ int ph_pad(int x) {
  using C = PhCfg<P>;
  if constexpr (C::DENSE) {
    return x;
  } else {
    const int row = x / (P * C::M), o = x - row * (P * C::M);
    const int i = row / P, j = row - i * P;
    return i * C::SI + j * C::SJ + o;
  }
}

// a dense [node][v] slice (global) into the padded slice buffer, asynchronous
// 8-byte copies, consecutive threads on consecutive doubles
template <int P, int NT>
__device__ __forceinline__ void ph_fetch(double* buf, const double* src, int tid) {
  using C = PhCfg<P>;
  for (int x = tid; x < (int)C::SLICE; x += NT) cp_async8(buf + ph_pad<P>(x), src + x);
  cp_async_commit();
}

// a stored (padded) slice of the iterate into the slice buffer: one bulk copy
// issued by thread 0, completion on the CTA's mbarrier.  Call after a
// __syncthreads() that ends every generic access to buf.
template <int P>
__device__ __forceinline__ void ph_fetch_bulk(double* buf, const double* src, uint64_t* bar,
                                              uint32_t& phase, int tid) {
  using C = PhCfg<P>;
  if (tid == 0) {
    fence_proxy_async_smem();
    mbar_expect_tx(bar, (uint32_t)(C::QSZP * 8));
    bulk_g2s(buf, src, (uint32_t)(C::QSZP * 8), bar);
  }
  mbar_wait(bar, phase);
  phase ^= 1u;
}

// rates of the slice in Q -> rt ([node][v], global): the owners contract their
// z line (partials published x-line-major in B), then their y line (added in
// place), then their x line: rate = -D_x F_x - (D_z F_z + D_y F_y).
// (Staging the slice of rates in shared memory for coalesced stores was
// measured neutral here: 8.26 vs 8.08 ms per sweep at N = 8, and it costs
// 30-50 registers.)
// OUT 0: rt is a dense [node][v] slice; OUT 1: a padded slice (the stored
// layout); OUT 2: padded, and the value stored is the rate minus the same
// thread's earlier OUT 1 output at sub (the startup's k2 - k1)
template <int P, int OUT>
__device__ __forceinline__ void ph_slice_rates(const double* Q, double* B, double* X,
                                               double* rt, const double* sub,
                                               const PhRoles<P>& R, bool owner, int half,
                                               double gm1, const double* dd, int tid) {
  using C = PhCfg<P>;
  constexpr int M = 5, H = C::H;
  const int ib = half * H;
  ph_prepass<P, C::NT_A>(Q, X, gm1, tid);
  double acc[H][M];
  if (owner) {
    ph_line<P, 2>(Q + R.qbase(2), R.qstride(2), X + 2 * R.nbase(2), 2 * R.nstride(2), gm1, dd,
                  half, acc);
    const int pb = R.pbase(2), ps = R.pstride(2);
#pragma unroll
    for (int i = 0; i < H; ++i)
      if (ib + i < P)
#pragma unroll
        for (int v = 0; v < M; ++v) B[pb + (ib + i) * ps + v] = acc[i][v];
  }
  __syncthreads();
  if (owner) {
    ph_line<P, 1>(Q + R.qbase(1), R.qstride(1), X + 2 * R.nbase(1), 2 * R.nstride(1), gm1, dd,
                  half, acc);
    const int pb = R.pbase(1), ps = R.pstride(1);
#pragma unroll
    for (int i = 0; i < H; ++i)
      if (ib + i < P)
#pragma unroll
        for (int v = 0; v < M; ++v) B[pb + (ib + i) * ps + v] += acc[i][v];
  }
  __syncthreads();
  if (owner) {
    ph_line<P, 0>(Q + R.qbase(0), R.qstride(0), X + 2 * R.nbase(0), 2 * R.nstride(0), gm1, dd,
                  half, acc);
    const int xr = R.xrow(), nb = R.nbase(0), ns = R.nstride(0);
    const int qb = R.qbase(0), qs = R.qstride(0);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      if (ib + i < P) {
        const int o = OUT == 0 ? (nb + (ib + i) * ns) * M : qb + (ib + i) * qs;
#pragma unroll
        for (int v = 0; v < M; ++v) {
          double val = -acc[i][v] - B[xr + (ib + i) * M + v];
          if (OUT == 2) val = val - sub[o + v];
          rt[o + v] = val;
        }
      }
    }
  }
}

// the startup iterate at time level t (predictor.py:116-124): q_t = u +
// s_t k1 + s_t^2 / (2 dt) (k2 - k1) from u, k1 and d = k2 - k1: one expression
// for every kernel that forms it
__device__ __forceinline__ double ph_startup_q(double un, double k1, double d, double s,
                                               double c2) {
  return fma(c2, d, fma(s, k1, un));
}

// ---------------------------------------------------------------- startup
// predictor.py:99-126: k1 = L(u), k2 = L(u + dt k1) into the element's K
// slices; the iterate itself is never stored (the first sweep's kernels form
// it from u, k1, k2).  Resets the element's state.
template <int P>
__global__ void __launch_bounds__(PhCfg<P>::NT_A, PhCfg<P>::MINB_A)
ph_startup_kernel(const __grid_constant__ PhArgs a) {
  using C = PhCfg<P>;
  constexpr int M = C::M, PP = C::PP, NW = C::NW;
  extern __shared__ __align__(16) double smem[];
  double* Q = smem;
  double* B = Q + C::QSZP;
  double* X = B + C::BSZP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = tid / C::RP, rr0 = tid - half * C::RP;
  const bool owner = rr0 < PP;
  const PhRoles<P> R(owner ? rr0 : 0);
  const double gm1 = a.gamma - 1.0;
  const double dt = *a.dt;
  for (int64_t e = blockIdx.x; e < a.n_elem; e += gridDim.x) {
    const double* ue = a.u + (size_t)e * C::SLICE;
    double* ke = a.kg + (size_t)e * 3 * C::QSZP;   // stored slices: u, k1, k2 - k1
    __syncthreads();   // previous element done with Q / B
    ph_fetch<P, C::NT_A>(Q, ue, tid);
    cp_async_wait_all();
    __syncthreads();
    for (int x = tid; x < C::QSZP; x += C::NT_A) ke[x] = Q[x];   // u in the stored layout
    ph_slice_rates<P, 1>(Q, B, X, ke + C::QSZP, nullptr, R, owner, half, gm1, a.dd, tid);   // k1
    __syncthreads();   // k1 stored, every line of Q read
    // w = u + dt k1 in the tile (k1 read back from this CTA's own stores)
    for (int x = tid; x < (int)C::SLICE; x += C::NT_A) {
      const int xp = ph_pad<P>(x);
      Q[xp] = Q[xp] + dt * ke[C::QSZP + xp];
    }
    __syncthreads();
    ph_slice_rates<P, 2>(Q, B, X, ke + 2 * C::QSZP, ke + C::QSZP, R, owner, half, gm1, a.dd,
                         tid);   // k2 - k1
    if (tid == 0) {
      a.state[e] = 0;
      a.state[a.n_elem + e] = 0;
      a.state[2 * a.n_elem + e] = 0;
      a.state[3 * a.n_elem + e] = 0;
      atomicAdd(a.n_active, 1);
    }
  }
}

// ------------------------------------------------------------------ rates
// one task per (element, time slice) of the elements still iterating; the
// first sweep (it == 0) forms its slice of the startup iterate from u, k1, k2
template <int P>
__global__ void __launch_bounds__(PhCfg<P>::NT_A, PhCfg<P>::MINB_A)
ph_rates_kernel(const __grid_constant__ PhArgs a) {
  using C = PhCfg<P>;
  constexpr int M = C::M, PP = C::PP, NW = C::NW;
  if (*a.n_active <= 0) return;
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double smem[];
  double* Q = smem;
  double* B = Q + C::QSZP;
  double* X = B + C::BSZP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = tid / C::RP, rr0 = tid - half * C::RP;
  const bool owner = rr0 < PP;
  const PhRoles<P> R(owner ? rr0 : 0);
  const double gm1 = a.gamma - 1.0;
  const double dt = *a.dt;
  const int64_t ntask = a.n_elem * P;
  __shared__ __align__(8) uint64_t bar;
  uint32_t phase = 0;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int64_t e = task / P;
    const int t = (int)(task - e * P);
    if (a.state[e]) continue;
    __syncthreads();   // previous task done with Q / B (first pass: barrier initialised)
    if (a.it == 0) {
      // the startup iterate's slice from the stored u, k1, k2 - k1: u and k1
      // land in Q and B by bulk copy while d travels through registers
      // (coalesced loads issued before the wait), one pass folds them
      const double s = T.nodes[t] * dt, c2 = 0.5 * s * s / dt;
      const double* ke = a.kg + (size_t)e * 3 * C::QSZP;
      if (tid == 0) {
        fence_proxy_async_smem();
        mbar_expect_tx(&bar, (uint32_t)(2 * C::QSZP * 8));
        bulk_g2s(Q, ke, (uint32_t)(C::QSZP * 8), &bar);
        bulk_g2s(B, ke + C::QSZP, (uint32_t)(C::QSZP * 8), &bar);
      }
      constexpr int NI = (C::QSZP + C::NT_A - 1) / C::NT_A;
      double dreg[NI];
#pragma unroll
      for (int k = 0; k < NI; ++k) {
        const int x = tid + k * C::NT_A;
        dreg[k] = x < C::QSZP ? __ldcs(ke + 2 * C::QSZP + x) : 0.0;
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int k = 0; k < NI; ++k) {
        const int x = tid + k * C::NT_A;
        if (x < C::QSZP) Q[x] = ph_startup_q(Q[x], B[x], dreg[k], s, c2);
      }
      __syncthreads();
    } else {
      ph_fetch_bulk<P>(Q, a.qg + (size_t)e * C::TILEQ + (size_t)t * C::QSZP, &bar, phase, tid);
    }
    ph_slice_rates<P, 0>(Q, B, X, a.rg + (size_t)e * C::TILE + (size_t)t * C::SLICE, nullptr, R,
                         owner, half, gm1, a.dd, tid);
  }
}

// ------------------------------------------------------------------- time
// predictor.py:175-185 over an element's P^3 m values: q_new(t) = dt sum_s
// gw[t][s] rate(s) + g0[t] u, residual norms (fixed-order block sum), the
// convergence test and per-element freezing; q <- q_new.  One CTA per
// element, one (node, quantity) per thread and pass: its P rates and P old
// iterates are loaded up front (all independent: HBM latency overlapped)
template <int P>
__global__ void __launch_bounds__(PhCfg<P>::NT_T, ADG_PH_TMINB)
ph_time_kernel(const __grid_constant__ PhArgs a) {
  using C = PhCfg<P>;
  constexpr int M = C::M, PD = C::PD, NT = C::NT_T, NW = NT / 32;
  if (*a.n_active <= 0) return;
  const DegreeTables& T = tab<P>();
  __shared__ double red[2 * NW];
  __shared__ double cst[2 * P];   // startup coefficients s_t, s_t^2 / (2 dt)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double dt = *a.dt;
  if (tid < P) {
    const double s = T.nodes[tid] * dt;
    cst[tid] = s;
    cst[P + tid] = 0.5 * s * s / dt;
  }
  __syncthreads();
  for (int64_t e = blockIdx.x; e < a.n_elem; e += gridDim.x) {
    if (a.state[e]) continue;
    const double* ue = a.u + (size_t)e * C::SLICE;
    const double* ke = a.kg + (size_t)e * 3 * C::QSZP;
    double* Qg = a.qg + (size_t)e * C::TILEQ;
    const double* Rg = a.rg + (size_t)e * C::TILE;
    double sd = 0.0, sq = 0.0;
    // NB items per thread in flight: their loads all issue before the first
    // use (the kernel is bound by HBM latency x bytes in flight)
    constexpr int NB = ADG_PH_TNB;
    for (int x0 = tid; x0 < PD * M; x0 += NB * NT) {
      double r[NB][P], qo[NB][P], uu[NB];
      int xp[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int x = x0 + b * NT < PD * M ? x0 + b * NT : x0;
        xp[b] = ph_pad<P>(x);   // position inside a stored (padded) slice
#pragma unroll
        for (int s2 = 0; s2 < P; ++s2) r[b][s2] = __ldcs(Rg + s2 * C::SLICE + x);
        uu[b] = ue[x];
        if (a.it == 0) {
          qo[b][0] = ke[C::QSZP + xp[b]];
          qo[b][1] = ke[2 * C::QSZP + xp[b]];
        } else {
#pragma unroll
          for (int t2 = 0; t2 < P; ++t2) qo[b][t2] = Qg[t2 * C::QSZP + xp[b]];
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (x0 + b * NT >= PD * M) break;
        if (a.it == 0) {
          const double k1 = qo[b][0], d = qo[b][1];
#pragma unroll
          for (int t2 = 0; t2 < P; ++t2)
            qo[b][t2] = ph_startup_q(uu[b], k1, d, cst[t2], cst[P + t2]);
        }
#pragma unroll
        for (int t2 = 0; t2 < P; ++t2) {
          double cc = 0.0;
#pragma unroll
          for (int s2 = 0; s2 < P; ++s2) cc = fma(T.gw[t2 * P + s2], r[b][s2], cc);
          const double qn = cc * dt + T.g0[t2] * uu[b];
          const double dq = qo[b][t2] - qn;
          sd = fma(dq, dq, sd);
          sq = fma(qn, qn, sq);
          Qg[t2 * C::QSZP + xp[b]] = qn;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sd += __shfl_xor_sync(0xffffffffu, sd, o);
      sq += __shfl_xor_sync(0xffffffffu, sq, o);
    }
    __syncthreads();   // previous element's readers of red are done
    if (lane == 0) {
      red[2 * warp] = sd;
      red[2 * warp + 1] = sq;
    }
    __syncthreads();
    if (tid == 0) {
      double t1 = 0.0, t2 = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        t1 += red[2 * w];
        t2 += red[2 * w + 1];
      }
      const double res = T.k1_opnorm * sqrt(t1);
      const double scale = 1.0 + sqrt(t2);
      const int c = res <= a.tol * scale;
      a.state[a.n_elem + e] = c;
      a.state[2 * a.n_elem + e] = a.it + 1;
      if ((c && a.it + 1 >= a.min_iter) || a.it + 1 >= a.max_iter) {
        a.state[e] = 1;
        atomicSub(a.n_active, 1);
      }
    }
  }
}

// ----------------------------------------------------------------- traces
// one task per (element, time slice): the 3 P^2 line owners extrapolate their
// line to both faces (predictor.py:218-230; face-kernel block layouts
// x [j][k][t][v], y [k][t][i][v], z [t][i][j][v]); optional q output
template <int P>
__global__ void __launch_bounds__(PhCfg<P>::NT_F, PhCfg<P>::MINB_TR)
ph_traces_kernel(const __grid_constant__ PhArgs a) {
  using C = PhCfg<P>;
  constexpr int M = C::M, PP = C::PP, PD = C::PD, NT = C::NT_F, NW = NT / 32;
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double smem[];
  double* Q = smem;
  double* S = Q + C::QSZP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = tid / C::RP;
  const int rr0 = tid - grp * C::RP;
  const bool owner = rr0 < PP;
  const int role = grp;
  const PhRoles<P> R(owner ? rr0 : 0);
  const int qbase = R.qbase(role), qstride = R.qstride(role);
  const int64_t ntask = a.n_elem * P;
  const size_t fs = (size_t)a.tr_elems * C::TB;
  // copy-out map of the staged traces, fixed per thread: entry k of this
  // thread is staged double x = tid + k NT; it lands at face f, block
  // position (base + t * tstride) * M + v
  constexpr int NC = (C::TRS + NT - 1) / NT;
  int cface[NC], cbase[NC], cstr[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int x = tid + k * NT < C::TRS ? tid + k * NT : 0;
    const int f = x / (PP * M);
    const int y = x - f * (PP * M);
    const int ln = y / M, v = y - ln * M;
    const int la = ln / P, lb = ln - la * P;
    const int rl = f >> 1;
    cface[k] = f;
    cbase[k] = (rl == 0 ? (la * P + lb) * P : (rl == 1 ? lb * P * P + la : la * P + lb)) * M + v;
    cstr[k] = (rl == 0 ? 1 : (rl == 1 ? P : P * P)) * M;
  }
  __shared__ __align__(8) uint64_t bar;
  uint32_t phase = 0;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {
    const int64_t e = task / P;
    const int t = (int)(task - e * P);
    __syncthreads();   // previous task done with Q / S
    ph_fetch_bulk<P>(Q, a.qg + (size_t)e * C::TILEQ + (size_t)t * C::QSZP, &bar, phase, tid);
    if (owner) {
      double lo[M], hi[M];
#pragma unroll
      for (int v = 0; v < M; ++v) lo[v] = hi[v] = 0.0;
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const double* src = Q + qbase + l * qstride;
        const double pl = T.left[l], pr = T.right[l];
#pragma unroll
        for (int v = 0; v < M; ++v) {
          lo[v] = fma(pl, src[v], lo[v]);
          hi[v] = fma(pr, src[v], hi[v]);
        }
      }
      double* slo = S + ((2 * role) * PP + rr0) * M;
#pragma unroll
      for (int v = 0; v < M; ++v) {
        slo[v] = lo[v];
        slo[PP * M + v] = hi[v];
      }
    }
    __syncthreads();
    // staged [face][line][v] -> the face blocks (x [j][k][t][v], y [k][t][i][v],
    // z [t][i][j][v]): consecutive threads write consecutive doubles of a
    // line's 40-byte block (z faces: one contiguous P^2 m run per slice)
    double* te = a.traces + (size_t)e * C::TB;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const int x = tid + k * NT;
      if (x < C::TRS) te[(size_t)cface[k] * fs + cbase[k] + t * cstr[k]] = S[x];
    }
    if (a.q_out) {
      for (int n = tid; n < PD; n += NT) {
        const int i = n / PP, j = (n / P) % P, k = n % P;
        const double* qn = Q + i * C::SI + j * C::SJ + k * M;
#pragma unroll
        for (int v = 0; v < M; ++v) a.q_out[(((size_t)e * PD + n) * P + t) * M + v] = qn[v];
      }
    }
  }
}

// ------------------------------------------------------------------- fbar
// streaming over the batch's nodes: admissibility of the final iterate
// (predictor.py:188-189) and the time-weighted fluxes Fbar_dir = sum_t w_t
// F_dir(q_t) (corrector.py:166) into the element's (now free) rate slices
// 0 / 1 / 2 = x / y / z, [node][v]
template <int P>
__global__ void __launch_bounds__(256, ADG_PH_FMINB)
ph_fbar_kernel(const __grid_constant__ PhArgs a) {
  using C = PhCfg<P>;
  constexpr int M = C::M, PD = C::PD;
  const DegreeTables& T = tab<P>();
  const double gm1 = a.gamma - 1.0;
  const int64_t total = a.n_elem * PD;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = g / PD;
    const int n = (int)(g - e * PD);
    const double* qe = a.qg + (size_t)e * C::TILEQ + ph_pad<P>(n * M);
    double fb[3][M];
    bool ok = true;
    // the next time level's state is loaded before this one is used (the
    // kernel waited on every level's load in turn: 59 % of its stall samples)
    double qn[M];
#pragma unroll
    for (int v = 0; v < M; ++v) qn[v] = qe[v];
#pragma unroll
    for (int t = 0; t < P; ++t) {
      double q[M];
#pragma unroll
      for (int v = 0; v < M; ++v) q[v] = qn[v];
      if (t + 1 < P) {
#pragma unroll
        for (int v = 0; v < M; ++v) qn[v] = qe[(size_t)(t + 1) * C::QSZP + v];
      }
      ok = admissible<3>(q, gm1) && ok;
      const double wt = T.weights[t];
      double f[M];
#pragma unroll
      for (int dir = 0; dir < 3; ++dir) {
        flux_axis<3>(q, gm1, dir, f);
#pragma unroll
        for (int v = 0; v < M; ++v) fb[dir][v] = t == 0 ? wt * f[v] : fb[dir][v] + wt * f[v];
      }
    }
    // (staged, coalesced stores were measured slower here: 2.87 vs 2.66 ms)
    double* re = a.rg + (size_t)e * C::TILE + (size_t)n * M;
#pragma unroll
    for (int dir = 0; dir < 3; ++dir)
#pragma unroll
      for (int v = 0; v < M; ++v) re[(size_t)dir * C::SLICE + v] = fb[dir][v];
    if (!ok) atomicOr(a.state + 3 * a.n_elem + e, 1);
  }
}

// -------------------------------------------------------------------- vol
// per element: one stiffness contraction per direction of its Fbar slices
// (corrector.py:169-176), y and z partials published x-line-major, the x-owner
// scales and sums; the element's flags leave with it
template <int P>
__device__ __forceinline__ void ph_stiff_line(const double* src0, int stride,
                                              const DegreeTables& T, double (&acc)[P][5]) {
  constexpr int M = 5;
#pragma unroll
  for (int i = 0; i < P; ++i)
#pragma unroll
    for (int v = 0; v < M; ++v) acc[i][v] = 0.0;
#pragma unroll 1
  for (int l = 0; l < P; ++l) {
    double f[M];
#pragma unroll
    for (int v = 0; v < M; ++v) f[v] = src0[l * stride + v];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const double d = T.stiff[i * P + l];
#pragma unroll
      for (int v = 0; v < M; ++v) acc[i][v] = fma(d, f[v], acc[i][v]);
    }
  }
}

template <int P>
__global__ void __launch_bounds__(PhCfg<P>::RP)
ph_vol_kernel(const __grid_constant__ PhArgs a) {
  using C = PhCfg<P>;
  constexpr int M = C::M, PP = C::PP, PD = C::PD, NW = C::RP / 32;
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double smem[];
  double* Q = smem;
  double* B1 = Q + C::QSZP;
  double* B2 = B1 + C::BSZP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool owner = tid < PP;
  const PhRoles<P> R(owner ? tid : 0);
  const int a0 = R.a0, b0 = R.b0;
  const double dt = *a.dt;
  const double cv = a.dx[0] * a.dx[1] * a.dx[2];
  const double sc0 = dt * cv / a.dx[0], sc1 = dt * cv / a.dx[1], sc2 = dt * cv / a.dx[2];
  for (int64_t e = blockIdx.x; e < a.n_elem; e += gridDim.x) {
    const double* fe = a.rg + (size_t)e * C::TILE;
    double acc[P][M];
#pragma unroll 1
    for (int role = 2; role >= 0; --role) {
      __syncthreads();   // previous readers of Q are done
      ph_fetch<P, C::RP>(Q, fe + (size_t)role * C::SLICE, tid);
      cp_async_wait_all();
      __syncthreads();
      if (owner) {
        ph_stiff_line<P>(Q + R.qbase(role), R.qstride(role), T, acc);
        if (role > 0) {
          double* pdst = role == 1 ? B1 : B2;
          const int pb = R.pbase(role), ps = R.pstride(role);
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int v = 0; v < M; ++v) pdst[pb + i * ps + v] = acc[i][v];
        }
      }
    }
    __syncthreads();   // partials published, every x line of Q read
    if (owner) {
      const int xrow = R.xrow(), nbase = R.nbase(0), nstride = R.nstride(0);
      const double wa = T.weights[a0], wb = T.weights[b0];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const double wi = T.weights[i];
        const double s0 = sc0 * (wa * wb), s1 = sc1 * (wi * wb), s2 = sc2 * (wi * wa);
        double* out = Q + (nbase + i * nstride) * M;   // node-major, unpadded
#pragma unroll
        for (int v = 0; v < M; ++v) {
          double vv = s0 * acc[i][v];
          vv += s1 * B1[xrow + i * M + v];
          vv += s2 * B2[xrow + i * M + v];
          out[v] = vv;
        }
      }
    }
    __syncthreads();
    {
      double* vole = a.vol + (size_t)e * PD * M;
      for (int x = tid; x < PD * M; x += C::RP) vole[x] = Q[x];
    }
    if (tid == 0) {
      const int conv = a.state[a.n_elem + e], nsw = a.state[2 * a.n_elem + e];
      const int bad = a.state[3 * a.n_elem + e];
      a.pred_bad[e] = (conv ? 0 : ADG_PRED_NOT_CONVERGED) | (bad ? ADG_PRED_INADMISSIBLE : 0);
      a.sweeps[e] = nsw;
    }
  }
}

// ------------------------------------------------------------------- host
template <int P>
static size_t phased_bytes_per_element() {
  return (PhCfg<P>::TILEQ + PhCfg<P>::TILE + 3 * PhCfg<P>::QSZP) * 8 + 4 * sizeof(int32_t);
}

// elements per batch: the whole grid, capped so the iterate + rates stay
// within kPhasedCapBytes
constexpr size_t kPhasedCapBytes = (size_t)28 << 30;

// ADG_PHASED_CAP_MB overrides the cap (tests force several batches with it)
static size_t phased_cap_bytes() {
  const char* c = getenv("ADG_PHASED_CAP_MB");
  const long mb = c ? atol(c) : 0;
  return mb > 0 ? (size_t)mb << 20 : kPhasedCapBytes;
}

template <int P>
static int64_t phased_batch(int64_t n_elem) {
  const int64_t cap = (int64_t)(phased_cap_bytes() / phased_bytes_per_element<P>());
  return std::max<int64_t>(1, std::min<int64_t>(n_elem, cap));
}

template <int P>
static size_t phased_ws_need(int64_t n_elem) {
  return (size_t)phased_batch<P>(n_elem) * phased_bytes_per_element<P>() + 256;
}

// per-device side stream + fork / join events of the two-stream schedule
struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream* side_stream() {
  static SideStream tab[32];
  int d = 0;
  cudaGetDevice(&d);
  SideStream* s = &tab[d & 31];
  if (!s->stream) {
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming) != cudaSuccess) {
      s->stream = nullptr;
      cudaGetLastError();
      return nullptr;
    }
  }
  return s;
}

template <class K>
static int set_smem(K kern, size_t bytes, PerDevice* flag, std::string* err) {
  if (!flag->first()) return ADG_OK;
  if (bytes <= 48 * 1024) return ADG_OK;
  cudaError_t ce =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

template <int P>
static int launch_phased(const PhArgs& a0, int64_t n_all, cudaStream_t st, int num_sms,
                         double* ws, size_t ws_bytes, std::string* err) {
  using C = PhCfg<P>;
  static PerDevice f_start, f_rates, f_tr, f_vol;
  int rc;
  if ((rc = set_smem(ph_startup_kernel<P>, C::SMEM_A, &f_start, err))) return rc;
  if ((rc = set_smem(ph_rates_kernel<P>, C::SMEM_A, &f_rates, err))) return rc;
  if ((rc = set_smem(ph_traces_kernel<P>, C::SMEM_TR, &f_tr, err))) return rc;
  if ((rc = set_smem(ph_vol_kernel<P>, C::SMEM_V, &f_vol, err))) return rc;
  const int64_t batch = phased_batch<P>(n_all);
  if (!ws || ws_bytes < phased_ws_need<P>(n_all)) {
    *err = "predictor workspace too small";
    return ADG_ERR_RUNTIME;
  }
  int occ_a = 1, occ_t = 1, occ_tr = 1, occ_v = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, ph_rates_kernel<P>, C::NT_A, C::SMEM_A);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, ph_time_kernel<P>, C::NT_T, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_tr, ph_traces_kernel<P>, C::NT_F,
                                                C::SMEM_TR);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_v, ph_vol_kernel<P>, C::RP, C::SMEM_V);
  occ_a = std::max(occ_a, 1);
  occ_t = std::max(occ_t, 1);
  occ_tr = std::max(occ_tr, 1);
  occ_v = std::max(occ_v, 1);
  // Two halves of a batch run their kernel sequences on two streams, the
  // second one kernel behind the first: the FP64-bound kernels (startup,
  // rates) of one half overlap the HBM-bound ones (time, traces, flux sums)
  // of the other (ADG_PH_STREAMS=1: one stream).  The side stream forks from
  // and joins the caller's stream by events (graph-capturable).
  const char* sv = getenv("ADG_PH_STREAMS");
  const int want_parts = sv ? atoi(sv) : 2;
  SideStream* side = want_parts > 1 ? side_stream() : nullptr;
  const auto grid = [&](int64_t tasks, int occ, int waves) {
    return (unsigned)std::max<int64_t>(1,
                                       std::min<int64_t>(tasks, (int64_t)num_sms * occ * waves));
  };
  for (int64_t e0 = 0; e0 < n_all; e0 += batch) {
    const int64_t n = std::min<int64_t>(batch, n_all - e0);
    const int nparts = (side && n >= 4 * (int64_t)num_sms) ? 2 : 1;
    double* qg = ws;
    // bulk-copied arrays first (16-byte aligned: QSZP is even), the dense
    // rates (odd slice sizes at P = 9) behind them
    double* kg = qg + (size_t)batch * C::TILEQ;
    double* rg = kg + 3 * (size_t)batch * C::QSZP;
    int32_t* state = reinterpret_cast<int32_t*>(rg + (size_t)batch * C::TILE);
    int32_t* n_active = state + 4 * batch;
    cudaMemsetAsync(n_active, 0, 2 * sizeof(int32_t), st);
    PhArgs part[2];
    cudaStream_t pst[2] = {st, nparts == 2 ? side->stream : st};
    for (int p = 0; p < nparts; ++p) {
      const int64_t off = p == 0 ? 0 : n / 2;
      const int64_t np = nparts == 1 ? n : (p == 0 ? n / 2 : n - n / 2);
      PhArgs& a = part[p];
      a = a0;
      a.u = a0.u + (size_t)(e0 + off) * C::SLICE;
      a.q_out = a0.q_out ? a0.q_out + (size_t)(e0 + off) * C::TILE : nullptr;
      a.vol = a0.vol + (size_t)(e0 + off) * C::SLICE;
      a.traces = a0.traces + (size_t)(e0 + off) * C::TB;
      a.pred_bad = a0.pred_bad + e0 + off;
      a.sweeps = a0.sweeps + e0 + off;
      a.n_elem = np;
      a.tr_elems = n_all;
      a.qg = qg + (size_t)off * C::TILEQ;
      a.kg = kg + 3 * (size_t)off * C::QSZP;
      a.rg = rg + (size_t)off * C::TILE;
      a.state = state + 4 * off;
      a.n_active = n_active + p;
    }
    if (nparts == 2) {
      cudaEventRecord(side->fork, st);
      cudaStreamWaitEvent(side->stream, side->fork, 0);
    }
    // kernel k of a part's sequence: 0 startup, 1 + 2 it rates, 2 + 2 it
    // time, then traces, flux sums, volume
    const int nk = 1 + 2 * a0.max_iter + 3;
    const auto launch = [&](int p, int k) {
      PhArgs& a = part[p];
      cudaStream_t s = pst[p];
      const int64_t np = a.n_elem;
      if (k == 0) {
        ph_startup_kernel<P><<<grid(np, occ_a, 4), C::NT_A, C::SMEM_A, s>>>(a);
      } else if (k <= 2 * a0.max_iter) {
        a.it = (k - 1) / 2;
        if (k & 1)
          ph_rates_kernel<P><<<grid(np * P, occ_a, 4), C::NT_A, C::SMEM_A, s>>>(a);
        else
          ph_time_kernel<P><<<grid(np, occ_t, 4), C::NT_T, 0, s>>>(a);
      } else if (k == nk - 3) {
        // (one fused per-element kernel for traces + flux sums, slices double
        // buffered by bulk copies, was measured equal: 6.18 vs 6.38 ms at N = 8)
        ph_traces_kernel<P><<<grid(np * P, occ_tr, 4), C::NT_F, C::SMEM_TR, s>>>(a);
      } else if (k == nk - 2) {
        ph_fbar_kernel<P><<<grid((np * C::PD + 255) / 256, 8, 4), 256, 0, s>>>(a);
      } else {
        ph_vol_kernel<P><<<grid(np, occ_v, 4), C::RP, C::SMEM_V, s>>>(a);
      }
    };
    const int lag = nparts == 2 ? 1 : 0;
    for (int k = 0; k < nk + lag; ++k)
      for (int p = 0; p < nparts; ++p) {
        const int kp = k - p * lag;
        if (kp >= 0 && kp < nk) launch(p, kp);
      }
    if (nparts == 2) {
      cudaEventRecord(side->join, side->stream);
      cudaStreamWaitEvent(st, side->join, 0);
    }
  }
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

bool predict_phased_supported(const adg_grid* g) {
  return g->dim == 3 && g->degree >= 7 && g->degree <= 9 && g->mode != ADG_MODE_PRIMITIVE;
}

size_t predict_phased_workspace_bytes(int P, int64_t n_elem) {
  switch (P) {
    case 8: return phased_ws_need<8>(n_elem);
    case 9: return phased_ws_need<9>(n_elem);
    case 10: return phased_ws_need<10>(n_elem);
  }
  return 0;
}

int predict_phased(const adg_grid* g, const double* u, const double* dt_dev, double tol,
                   int max_iter, int min_iter, double* q_out, double* vol, double* traces,
                   uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms, double* ws,
                   size_t ws_bytes, std::string* err) {
  PhArgs a{};
  a.u = u;
  a.dt = dt_dev;
  a.q_out = q_out;
  a.vol = vol;
  a.traces = traces;
  a.pred_bad = pred_bad;
  a.sweeps = sweeps;
  const int64_t n_all = g->cells[0] * g->cells[1] * g->cells[2];
  for (int j = 0; j < 3; ++j) a.dx[j] = g->dx[j];
  a.gamma = g->gamma;
  a.tol = tol;
  a.max_iter = max_iter > 0 ? max_iter : 2 * g->degree + 2;
  a.min_iter = min_iter;
  const int P = g->degree + 1;
  for (int dir = 0; dir < 3; ++dir)
    for (int x = 0; x < P * P; ++x) a.dd[dir * P * P + x] = h_tab[g->degree].diff[x] / g->dx[dir];
  if (n_all < 1) return ADG_OK;
  switch (P) {
    case 8: return launch_phased<8>(a, n_all, st, num_sms, ws, ws_bytes, err);
    case 9: return launch_phased<9>(a, n_all, st, num_sms, ws, ws_bytes, err);
    case 10: return launch_phased<10>(a, n_all, st, num_sms, ws, ws_bytes, err);
  }
  *err = "phased predictor: unsupported degree";
  return ADG_ERR_UNSUPPORTED;
}

}  // namespace adg
