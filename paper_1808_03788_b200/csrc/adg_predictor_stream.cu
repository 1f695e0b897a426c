// adg_predictor_stream.cu -- the fused ADER-DG predictor for the large 3-D
// space-time tiles (P = N+1 = 8..10: 160-391 KB per element, more than one
// SM's shared memory) as a slice-streaming kernel: one CTA per element, the
// element's space-time iterate and rates in a per-CTA global scratch that
// stays in L2, one time slice at a time in shared memory.
//
// Same algorithm and outputs as predict_kernel (adg_predictor.cu): startup
// guess (predictor.py:99-126), Picard sweeps with per-element freezing
// (predictor.py:135-191), admissibility (:188-189), face traces (:218-230)
// and the volume integral (corrector.py:141-177).
//
// The Picard rate L(q_t) = -sum_dir D_dir F_dir(q_t) only couples the nodes of
// one time slice, and the time operator q_new = dt gw (x)_t rate + g0 (x) u
// only couples the time levels of one spatial node.  So a sweep is
//   (1) for t = 0..P-1: slice t of q -> shared memory (cp.async; the next
//       slice is fetched while the current slice's rates are stored), the
//       3 P^2 line owners contract the slice's flux lines, and
//       the x-owner stores the slice's rates to the scratch;
//   (2) node phase: every thread takes nodes n, reads rate[0..P-1][n] (P x m
//       values in registers), forms q_new at every time, the residual
//       partials and stores q_new over q.
// All CTAs of the GPU stay busy on their own element; the slice buffers use
// conflict-light padded layouts (tools/slice_bankcheck.py).  The startup guess needs only two
// spatial passes on u (k1 = L(u), k2 = L(u + dt k1)); the q at every time is a
// pointwise formula of (u, k1, k2).
#include <algorithm>
#include <type_traits>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

#ifndef ADG_STREAM_LUNROLL
#define ADG_STREAM_LUNROLL 1
#endif
#ifndef ADG_STREAM_NH
#define ADG_STREAM_NH 0   // 0: per-degree default below; 1 / 2: force
#endif

#ifndef ADG_STREAM_DBUF
#define ADG_STREAM_DBUF 0   // 1: second slice buffer (measured neutral: C3 N=7..9 within 1 %)
#endif

template <int P>
struct StCfg {
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
  static constexpr int BSZP = BSZ + (BSZ & 1);
  // output halves per line: with NH = 2 two warp groups own the same lines,
  // each recomputes the line's fluxes and accumulates half of the P outputs
  // (P x m accumulators do not fit the register budget at P >= 9)
  static constexpr int NH = ADG_STREAM_NH ? ADG_STREAM_NH : 1;
  static constexpr int H = (P + NH - 1) / NH;
  // warp-aligned line groups: every warp contracts along one compile-time
  // direction and half (D/dx coefficients as constant-bank operands, no
  // divergence)
  static constexpr int RP = ((PP + 31) / 32) * 32;
  static constexpr int NG = 3 * NH;
  static constexpr int NT = NG * RP;
  static constexpr int NW = NT / 32;
  static constexpr int CSTP = (2 * P + 1) / 2 * 2;  // startup coefficients, padded to 16 B
  // two slice buffers (the next slice lands while the current one is contracted)
  static constexpr int NQB = ADG_STREAM_DBUF ? 2 : 1;
  static constexpr size_t SMEM = (NQB * (size_t)QSZP + 2 * (size_t)BSZP + 2 * NW + CSTP) * 8;
  // CTAs per SM: what shared memory allows, capped so each thread keeps
  // >= 80 registers (H x m accumulators)
  static constexpr int MINB0 = (int)((228 * 1024) / (SMEM + 1024));
#ifndef ADG_STREAM_RMIN
#define ADG_STREAM_RMIN 168
#endif
  static constexpr int RMIN = NH == 1 ? ADG_STREAM_RMIN : 80;
  static constexpr int MINB_R = 65536 / (RMIN * NT) > 0 ? 65536 / (RMIN * NT) : 1;
  static constexpr int MINB1 = MINB0 < MINB_R ? MINB0 : MINB_R;
  static constexpr int MINB = MINB1 < 1 ? 1 : MINB1;
  static constexpr int TB = PD * M + ((PD * M) & 1);   // trace block (face kernel layout)
  static constexpr size_t SLICE = (size_t)PD * M;      // doubles per time slice
  // the iterate's slices sit in the scratch in the PADDED shared layout (QSZP
  // doubles, even), so a slice is one 16-byte-aligned bulk copy (TMA) into Q
  // instead of P^3 m 8-byte cp.async (ADG_STREAM_BULK=0: dense slices)
#ifndef ADG_STREAM_BULK
#define ADG_STREAM_BULK 1
#endif
  static constexpr bool BULK = ADG_STREAM_BULK;
  static constexpr size_t QSL = BULK ? (size_t)QSZP : SLICE;   // stored slice stride
  static constexpr size_t SCR0 = (size_t)P * QSL + (size_t)P * SLICE;   // q + rates per CTA
  static constexpr size_t SCR = SCR0 + (SCR0 & 1);
};

struct StArgs {
  const double* u;
  const double* dt;
  double* q_out;
  double* vol;
  double* traces;
  uint8_t* pred_bad;
  int32_t* sweeps;
  double* scr;          // per-CTA [q: P slices][rates: P slices], slice = [node][v]
  int64_t n_elem;
  double dx[3];
  double gamma;
  double tol;
  int max_iter;
  int min_iter;
  double dd[3 * kMaxP * kMaxP];   // D / dx_dir, [dir][P][P] (kernel-parameter constant bank)
};

// one line's P states (src + l * stride) -> flux along DIR -> the outputs
// HF * H .. HF * H + H - 1 of the P x P contraction, l-outer (MODE 0: D/dx_DIR
// from the kernel-parameter bank; MODE 1: the stiffness, plus the
// admissibility screen)
template <int P, int DIR, int MODE, int HF>
__device__ __forceinline__ void st_line(const double* src0, int stride, double gm1,
                                        const double* dd, const DegreeTables& T,
                                        double (&acc)[StCfg<P>::H][5], bool& ok) {
  constexpr int M = 5, H = StCfg<P>::H, IB = HF * H;
#pragma unroll
  for (int i = 0; i < H; ++i)
#pragma unroll
    for (int v = 0; v < M; ++v) acc[i][v] = 0.0;
  // l unrolled by ADG_STREAM_LUNROLL (1: one source node's flux live at a
  // time next to the accumulators)
  constexpr int LU = ADG_STREAM_LUNROLL;
#pragma unroll LU
  for (int l = 0; l < P; ++l) {
    double q[M], f[M];
    const double* src = src0 + l * stride;
#pragma unroll
    for (int v = 0; v < M; ++v) q[v] = src[v];
    if (DIR >= 0) {
      flux_axis<3>(q, gm1, DIR < 0 ? 0 : DIR, f);
    } else {
#pragma unroll
      for (int v = 0; v < M; ++v) f[v] = q[v];   // precomputed (time-weighted) fluxes
    }
    if (MODE == 1 && DIR >= 0) ok = ok && admissible<3>(q, gm1);
#pragma unroll
    for (int ii = 0; ii < H; ++ii) {
      if (IB + ii < P) {
        const double d = MODE == 0 ? dd[(DIR < 0 ? 0 : DIR) * P * P + (IB + ii) * P + l] : T.stiff[(IB + ii) * P + l];
#pragma unroll
        for (int v = 0; v < M; ++v) acc[ii][v] = fma(d, f[v], acc[ii][v]);
      }
    }
  }
}

template <int P, int DIR, int MODE>
__device__ __forceinline__ void st_line_half(const double* src0, int stride, double gm1,
                                             const double* dd, const DegreeTables& T, int half,
                                             double (&acc)[StCfg<P>::H][5], bool& ok) {
  if (StCfg<P>::NH == 1 || half == 0)
    st_line<P, DIR, MODE, 0>(src0, stride, gm1, dd, T, acc, ok);
  else
    st_line<P, DIR, MODE, StCfg<P>::NH - 1>(src0, stride, gm1, dd, T, acc, ok);
}

// register budget: a CTA's warps are spread over the SM's four 16K-register
// sub-partitions, so 9 or 12 warps (P = 9, 10) allow at most 168 registers
// per thread, and P >= 9 spill the P x m line accumulators there (~1 KB per
// thread).  ADG_STREAM_MAXNREG sets the cap explicitly for A/B builds
// (profiles/r02_stream_regs.md: more registers cost P = 8 its second CTA per
// SM, and P = 9 / 10 cannot launch above 168)
#ifdef ADG_STREAM_MAXNREG
// (P = 8 keeps the launch bounds: two CTAs per SM at 168 registers)
#define ADG_STREAM_ATTR                                                               \
  __maxnreg__(P == 8 ? 168                                                            \
                     : ((ADG_STREAM_MAXNREG < (65536 / StCfg<P>::NT) / 8 * 8 - 8)     \
                            ? ADG_STREAM_MAXNREG                                      \
                            : (65536 / StCfg<P>::NT) / 8 * 8 - 8))
#else
#define ADG_STREAM_ATTR __launch_bounds__(StCfg<P>::NT, StCfg<P>::MINB)
#endif
template <int P>
__global__ void ADG_STREAM_ATTR
predict_stream_kernel(const __grid_constant__ StArgs a) {
  using C = StCfg<P>;
  constexpr int M = C::M, PP = C::PP, PD = C::PD, NT = C::NT, NW = C::NW, H = C::H, NH = C::NH;
  constexpr int SI = C::SI, SJ = C::SJ, TJ = C::TJ, TK = C::TK;
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double smem[];
  double* Q = smem;                 // current slice tile, node-major (padded)
  double* B1 = Q + C::QSZP;         // y partials (x-line-major, padded)
  double* B2 = B1 + C::BSZP;        // z partials (x-line-major)
  double* red = B2 + C::BSZP;       // [NW][2] warp partials
  double* cst = red + 2 * NW;       // startup coefficients [P] s_t = tau_t dt, [P] s_t^2 / (2 dt)
  double* const Qa = Q;             // the two slice buffers; Q is the current one
  double* const Qb = C::NQB == 2 ? cst + C::CSTP : Qa;
  double* Qg = a.scr + (size_t)blockIdx.x * C::SCR;   // q[t][node][v]
  double* Rg = Qg + P * C::QSL;                        // rate[t][node][v]; k1 at startup

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const double gm1 = a.gamma - 1.0;
  const double dt = *a.dt;

  // line ownership: group g = (direction, half); lanes rr >= P^2 of a group
  // are idle in the line phases
  const int grp = tid / C::RP;
  const int rr0 = tid - grp * C::RP;
  const bool owner = rr0 < PP;
  const int role = owner ? grp / NH : 3;      // 0/1/2 = x/y/z line, 3 idle
  const int half = grp - (grp / NH) * NH;     // output half (warp-uniform)
  const int ibase = half * H;                 // first output of this half
  const int rr = owner ? rr0 : 0;
  const int a0 = rr / P, b0 = rr - (rr / P) * P;
  const int qbase = role == 0 ? a0 * SJ + b0 * M : (role == 1 ? a0 * SI + b0 * M : a0 * SI + b0 * SJ);
  const int qstride = role == 0 ? SI : (role == 1 ? SJ : M);
  const int nbase = role == 0 ? a0 * P + b0 : (role == 1 ? a0 * PP + b0 : a0 * PP + b0 * P);
  const int nstride = role == 0 ? PP : (role == 1 ? P : 1);
  const int pbase = role == 1 ? b0 * TK + a0 * M : b0 * TJ + a0 * M;
  const int pstride = role == 1 ? TJ : TK;
  double* pdst = role == 1 ? B1 : B2;
  const int xrow = a0 * TJ + b0 * TK;     // x-owner's row in B1/B2

  const double cv = a.dx[0] * a.dx[1] * a.dx[2];
  const double sc0 = dt * cv / a.dx[0], sc1 = dt * cv / a.dx[1], sc2 = dt * cv / a.dx[2];

  if (tid < P) {
    const double s = T.nodes[tid] * dt;
    cst[tid] = s;
    cst[P + tid] = 0.5 * s * s / dt;
  }
  // (visible after the element loop's first barrier)

  auto line_contract = [&](int mode, double (&acc)[H][M], bool& ok) {
    const double* q0 = Q + qbase;
    if (mode == 0) {
      if (role == 0) st_line_half<P, 0, 0>(q0, qstride, gm1, a.dd, T, half, acc, ok);
      else if (role == 1) st_line_half<P, 1, 0>(q0, qstride, gm1, a.dd, T, half, acc, ok);
      else st_line_half<P, 2, 0>(q0, qstride, gm1, a.dd, T, half, acc, ok);
    } else {
      if (role == 0) st_line_half<P, 0, 1>(q0, qstride, gm1, a.dd, T, half, acc, ok);
      else if (role == 1) st_line_half<P, 1, 1>(q0, qstride, gm1, a.dd, T, half, acc, ok);
      else st_line_half<P, 2, 1>(q0, qstride, gm1, a.dd, T, half, acc, ok);
    }
  };
  auto publish = [&](const double (&acc)[H][M]) {
#pragma unroll
    for (int ii = 0; ii < H; ++ii)
      if (ibase + ii < P)
#pragma unroll
        for (int v = 0; v < M; ++v) pdst[pbase + (ibase + ii) * pstride + v] = acc[ii][v];
  };
  // a [node][v] slice (global) into the padded Q (asynchronous 8-byte copies)
  auto fetch_to = [&](double* buf, const double* src) {
    // P^2 rows (i, j) of P m contiguous doubles; one warp per row
    for (int row = warp; row < PP; row += NW) {
      const int i = row / P, j = row - (row / P) * P;
      double* dst = buf + i * SI + j * SJ;
      const double* sr = src + row * (P * M);
      for (int o = lane; o < P * M; o += 32) cp_async8(dst + o, sr + o);
    }
    cp_async_commit();
  };
  auto fetch = [&](const double* src) { fetch_to(Q, src); };
  // position of the x-th double of a dense [node][v] slice inside a stored slice
  auto spad = [&](int x) {
    if (!C::BULK) return x;
    const int row = x / (P * M), o = x - row * (P * M);
    const int i = row / P, j = row - i * P;
    return i * SI + j * SJ + o;
  };
  // a stored slice -> Q by one bulk copy (thread 0, after a barrier that ends
  // every access to Q; the scratch writers fenced their stores for the async
  // proxy); completion on the CTA's mbarrier
  __shared__ __align__(8) uint64_t bar;
  uint32_t bphase = 0;
  bool bulk_pending = false;   // uniform: the fetch in flight is a bulk copy
  if (C::BULK && tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  auto fetch_slice_to = [&](double* buf, const double* src) {
    if (C::BULK) {
      if (tid == 0) {
        fence_proxy_async_smem();
        mbar_expect_tx(&bar, (uint32_t)(C::QSZP * 8));
        bulk_g2s(buf, src, (uint32_t)(C::QSZP * 8), &bar);
      }
      bulk_pending = true;
    } else {
      fetch_to(buf, src);
    }
  };
  auto fetch_slice = [&](const double* src) { fetch_slice_to(Q, src); };
  auto wait_fetch = [&]() {
    if (C::BULK && bulk_pending) {
      mbar_wait(&bar, bphase);
      bphase ^= 1u;
      bulk_pending = false;
    } else {
      cp_async_wait_all();
    }
  };
  // fixed-order block sum of two partials (warp trees, warps in order)
  auto block_sum2 = [&](double& s1, double& s2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      red[2 * warp] = s1;
      red[2 * warp + 1] = s2;
    }
    __syncthreads();
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      t1 += red[2 * w];
      t2 += red[2 * w + 1];
    }
    s1 = t1;
    s2 = t2;
  };

  // rates of the slice in Q at the line owners' nodes -> rt ([node][v]);
  // the next slice (if any) is fetched into the other buffer meanwhile
  auto slice_rates = [&](const double* next, double* rt) {
    wait_fetch();
    __syncthreads();
    // the other buffer held the previous slice (its readers passed the
    // barrier above): the next slice lands there during this contraction
    double* const Qn = Q == Qa ? Qb : Qa;
    if (C::NQB == 2 && next) fetch_slice_to(Qn, next);
    double acc[H][M];
    bool dummy = true;
    if (owner) line_contract(0, acc, dummy);
    if (role == 1 || role == 2) publish(acc);
    __syncthreads();
    if (C::NQB == 1 && next) fetch_slice(next);   // single buffer: Q is dead now
    if (role == 0) {
#pragma unroll
      for (int ii = 0; ii < H; ++ii) {
        const int i = ibase + ii;
        if (i >= P) continue;
        const int n = nbase + i * nstride;
#pragma unroll
        for (int v = 0; v < M; ++v)
          rt[n * M + v] = (-acc[ii][v] - B1[xrow + i * M + v]) - B2[xrow + i * M + v];
      }
    }
    if (next) Q = Qn;
  };

  // time operator of the sweep (predictor.py:175-185) over the element's
  // P^3 m values: q_new(t) = dt sum_s gw[t][s] rate(s) + g0[t] u, residual
  // partials, q <- q_new.  Two items per thread in flight: their 2P rates and
  // 2P iterates are loaded before any arithmetic (L2 latency overlapped)
  auto node_phase = [&](const double* ue, double& sd, double& sq) {
    constexpr int NB = 2;
    for (int x0 = tid; x0 < PD * M; x0 += NB * NT) {
      double r[NB][P], qo[NB][P], uu[NB];
      int xp[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int x = x0 + b * NT < PD * M ? x0 + b * NT : x0;
        xp[b] = spad(x);
#pragma unroll
        for (int s2 = 0; s2 < P; ++s2) r[b][s2] = Rg[s2 * C::SLICE + x];
#pragma unroll
        for (int t2 = 0; t2 < P; ++t2) qo[b][t2] = Qg[t2 * C::QSL + xp[b]];
        uu[b] = ue[x];
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int x = x0 + b * NT;
        if (x >= PD * M) break;
#pragma unroll
        for (int t2 = 0; t2 < P; ++t2) {
          double cc = 0.0;
#pragma unroll
          for (int s2 = 0; s2 < P; ++s2) cc = fma(T.gw[t2 * P + s2], r[b][s2], cc);
          const double qn = cc * dt + T.g0[t2] * uu[b];
          const double dq = qo[b][t2] - qn;
          sd = fma(dq, dq, sd);
          sq = fma(qn, qn, sq);
          Qg[t2 * C::QSL + xp[b]] = qn;
        }
      }
    }
    if (C::BULK) asm volatile("fence.proxy.async;" ::: "memory");   // stores -> bulk reads
  };

  for (int64_t e = blockIdx.x; e < a.n_elem; e += gridDim.x) {
    const double* ue = a.u + (size_t)e * PD * M;
    __syncthreads();   // previous element's readers of Q / B / red are done
    int it = 0, conv = 0, nsw = 0;
    // ---------------- startup guess and Picard sweeps --------------------
    // one slice-rate call site for both (a second inlined copy spills):
    // stage 0 / 1 are the startup passes k1 = L(u), k2 = L(u + dt k1)
    // (predictor.py:99-126) on the tile in Q, stage 2 the sweeps' slices
    fetch(ue);
    bool fz = a.max_iter <= 0;
    int stage = 0, t = 0;
#pragma unroll 1
    while (true) {
      double* rt = Rg + (stage < 2 ? stage : t) * C::SLICE;
      const double* next = (stage == 2 && t + 1 < P) ? Qg + (t + 1) * C::QSL : nullptr;
      slice_rates(next, rt);
      if (stage == 0) {
        __syncthreads();   // k1 stored
        // w = u + dt k1 in the tile (row-parallel, like fetch)
        for (int row = warp; row < PP; row += NW) {
          const int i = row / P, j = row - (row / P) * P;
          double* dst = Q + i * SI + j * SJ;
          const double* k1 = Rg + row * (P * M);
          for (int o = lane; o < P * M; o += 32) dst[o] = dst[o] + dt * k1[o];
        }
        stage = 1;
        continue;
      }
      if (stage == 1) {
        __syncthreads();   // k2 stored
        // q_t = u + s_t k1 + s_t^2 / (2 dt) (k2 - k1) at every time (predictor.py:116-124)
        for (int x = tid; x < PD * M; x += NT) {
          const double k1 = Rg[x], k2 = Rg[C::SLICE + x], un = ue[x];
          const int xq = spad(x);
#pragma unroll 1
          for (int tt = 0; tt < P; ++tt)
            Qg[tt * C::QSL + xq] = un + cst[tt] * k1 + cst[P + tt] * (k2 - k1);
        }
        if (C::BULK) asm volatile("fence.proxy.async;" ::: "memory");   // stores -> bulk reads
        if (fz) break;
        stage = 2;
        t = 0;
        __syncthreads();   // startup iterate stored
        fetch_slice(Qg);
        continue;
      }
      if (++t < P) continue;
      __syncthreads();   // every slice's rates stored
      // node phase: time operator, residual partials, q <- q_new (one
      // quantity of one node per item: its P rates and P iterates loaded
      // up front)
      double sd = 0.0, sq = 0.0;
      node_phase(ue, sd, sq);
      block_sum2(sd, sq);
      const double res = T.k1_opnorm * sqrt(sd);
      const double scale = 1.0 + sqrt(sq);
      conv = res <= a.tol * scale;
      nsw = it + 1;
      ++it;
      if (conv && it >= a.min_iter) fz = true;
      if (fz || it >= a.max_iter) break;
      t = 0;
      __syncthreads();   // node-phase stores visible
      fetch_slice(Qg);
    }

    // ---------------- traces, admissibility, volume ---------------------
    // per slice: face traces (line owners), admissibility and the
    // time-weighted fluxes Fbar_dir = sum_t w_t F_dir(q_t) (corrector.py:166,
    // one node per thread: Fbar_y / Fbar_z accumulate in B1 / B2 in x-line-
    // major order, Fbar_x in the thread's own scratch rows); then one
    // stiffness contraction per direction (corrector.py:169-176)
    bool ok = true;
    constexpr int NPT = (PD + NT - 1) / NT;   // nodes per thread
    double fbx[NPT][M];                        // Fbar_x of the thread's nodes
    __syncthreads();   // node-phase stores of the final iterate visible
    fetch_slice(Qg);
#pragma unroll 1
    for (int t = 0; t < P; ++t) {
      wait_fetch();
      __syncthreads();
      if (owner && half == 0) {
        // face traces of the line at time t (face-kernel block layouts:
        // x [j][k][t][v], y [k][t][i][v], z [t][i][j][v])
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
        const int dir = role;
        const int pos = role == 0 ? (a0 * P + b0) * P + t
                                  : (role == 1 ? (b0 * P + t) * P + a0 : (t * P + a0) * P + b0);
        const size_t fs = (size_t)a.n_elem * C::TB;
        double* tlo = a.traces + (size_t)(2 * dir) * fs + (size_t)e * C::TB + (size_t)pos * M;
        double* thi = tlo + fs;
#pragma unroll
        for (int v = 0; v < M; ++v) {
          tlo[v] = lo[v];
          thi[v] = hi[v];
        }
      }
      const double wt = T.weights[t];
#pragma unroll
      for (int kk = 0; kk < NPT; ++kk) {
        const int n = tid + kk * NT;
        if (n >= PD) break;
        const int i = n / PP, j = (n / P) % P, k = n % P;
        const double* qn = Q + i * SI + j * SJ + k * M;
        double q[M];
#pragma unroll
        for (int v = 0; v < M; ++v) q[v] = qn[v];
        ok = ok && admissible<3>(q, gm1);
        if (a.q_out) {
#pragma unroll
          for (int v = 0; v < M; ++v) a.q_out[(((size_t)e * PD + n) * P + t) * M + v] = q[v];
        }
        double f[M];
        const int bx = j * TJ + k * TK + i * M;
        flux_axis<3>(q, gm1, 0, f);
#pragma unroll
        for (int v = 0; v < M; ++v) fbx[kk][v] = t == 0 ? wt * f[v] : fbx[kk][v] + wt * f[v];
        flux_axis<3>(q, gm1, 1, f);
#pragma unroll
        for (int v = 0; v < M; ++v) B1[bx + v] = t == 0 ? wt * f[v] : B1[bx + v] + wt * f[v];
        flux_axis<3>(q, gm1, 2, f);
#pragma unroll
        for (int v = 0; v < M; ++v) B2[bx + v] = t == 0 ? wt * f[v] : B2[bx + v] + wt * f[v];
      }
      __syncthreads();
      if (t + 1 < P) fetch_slice(Qg + (t + 1) * C::QSL);
    }
    // Fbar_x into Q (own nodes); the y / z owners contract Fbar_y / Fbar_z
    // in place (each reads and writes only its own line of B1 / B2)
#pragma unroll
    for (int kk = 0; kk < NPT; ++kk) {
      const int n = tid + kk * NT;
      if (n >= PD) break;
      const int i = n / PP, j = (n / P) % P, k = n % P;
#pragma unroll
      for (int v = 0; v < M; ++v) Q[i * SI + j * SJ + k * M + v] = fbx[kk][v];
    }
    __syncthreads();
    {
      double acc[H][M];
      bool dummy = true;
      if (owner) {
        const double* src0 = role == 0 ? Q + qbase : pdst + pbase;
        const int str = role == 0 ? qstride : pstride;
        st_line_half<P, -1, 1>(src0, str, gm1, a.dd, T, half, acc, dummy);
      }
      if (role == 1 || role == 2) publish(acc);
      __syncthreads();
      if (role == 0) {
        double* vole = a.vol + (size_t)e * PD * M;
        const double wa = T.weights[a0], wb = T.weights[b0];
#pragma unroll
        for (int ii = 0; ii < H; ++ii) {
          const int i = ibase + ii;
          if (i >= P) continue;
          const double wi = T.weights[i];
          const double s0 = sc0 * (wa * wb), s1 = sc1 * (wi * wb), s2 = sc2 * (wi * wa);
          double* out = vole + (nbase + i * nstride) * M;
#pragma unroll
          for (int v = 0; v < M; ++v) {
            double vv = s0 * acc[ii][v];
            vv += s1 * B1[xrow + i * M + v];
            vv += s2 * B2[xrow + i * M + v];
            out[v] = vv;
          }
        }
      }
    }
    const int all_ok = __syncthreads_and(ok ? 1 : 0);
    if (tid == 0) {
      a.pred_bad[e] = (conv ? 0 : ADG_PRED_NOT_CONVERGED) | (all_ok ? 0 : ADG_PRED_INADMISSIBLE);
      a.sweeps[e] = nsw ? nsw : it;
    }
  }
}

template <int P>
static size_t stream_ws_need(int num_sms) {
  using C = StCfg<P>;
  return (size_t)num_sms * C::MINB * C::SCR * 8;
}

template <int P>
static int launch_stream(const StArgs& a0, cudaStream_t st, int num_sms, double* ws,
                         size_t ws_bytes, std::string* err) {
  using C = StCfg<P>;
  auto kern = predict_stream_kernel<P>;
  static PerDevice attr;
  if (attr.first()) {
    cudaError_t ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)C::SMEM);
    if (ce != cudaSuccess) {
      *err = cudaGetErrorString(ce);
      return ADG_ERR_CUDA;
    }
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::NT, C::SMEM);
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)(ws_bytes / (C::SCR * 8));
  const int64_t grid = std::min<int64_t>(a0.n_elem, std::min<int64_t>(cap, (int64_t)num_sms * per_sm));
  if (a0.n_elem < 1) return ADG_OK;
  if (grid < 1 || !ws) {
    *err = "predictor workspace too small";
    return ADG_ERR_RUNTIME;
  }
  StArgs a = a0;
  a.scr = ws;
  kern<<<(unsigned)grid, C::NT, C::SMEM, st>>>(a);
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  return ADG_OK;
}

bool predict_stream_supported(const adg_grid* g) {
  return g->dim == 3 && g->degree >= 7 && g->degree <= 9 && g->mode != ADG_MODE_PRIMITIVE;
}

size_t predict_stream_workspace_bytes(int P, int num_sms) {
  switch (P) {
    case 8: return stream_ws_need<8>(num_sms);
    case 9: return stream_ws_need<9>(num_sms);
    case 10: return stream_ws_need<10>(num_sms);
  }
  return 0;
}

int predict_stream(const adg_grid* g, const double* u, const double* dt_dev, double tol,
                   int max_iter, int min_iter, double* q_out, double* vol, double* traces,
                   uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms, double* ws,
                   size_t ws_bytes, std::string* err) {
  StArgs a{};
  a.u = u;
  a.dt = dt_dev;
  a.q_out = q_out;
  a.vol = vol;
  a.traces = traces;
  a.pred_bad = pred_bad;
  a.sweeps = sweeps;
  a.n_elem = g->cells[0] * g->cells[1] * g->cells[2];
  for (int j = 0; j < 3; ++j) a.dx[j] = g->dx[j];
  a.gamma = g->gamma;
  a.tol = tol;
  a.max_iter = max_iter > 0 ? max_iter : 2 * g->degree + 2;
  a.min_iter = min_iter;
  const int P = g->degree + 1;
  for (int dir = 0; dir < 3; ++dir)
    for (int x = 0; x < P * P; ++x) a.dd[dir * P * P + x] = h_tab[g->degree].diff[x] / g->dx[dir];
  switch (P) {
    case 8: return launch_stream<8>(a, st, num_sms, ws, ws_bytes, err);
    case 9: return launch_stream<9>(a, st, num_sms, ws, ws_bytes, err);
    case 10: return launch_stream<10>(a, st, num_sms, ws, ws_bytes, err);
  }
  *err = "stream predictor: unsupported degree";
  return ADG_ERR_UNSUPPORTED;
}

}  // namespace adg
