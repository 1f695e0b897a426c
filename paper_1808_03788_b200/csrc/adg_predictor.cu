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
// Shared memory is the bottleneck resource of this kernel (16 doubles per
// clock per SM; for 64-bit accesses a broadcast does not save wavefronts),
// so the schedule minimises shared doubles moved per thread.  A Picard
// sweep (P = N+1 nodes per axis, m quantities) is
//   A  x-owner (x-line, time t): loads its line of q, F_x on its P nodes,
//      -D_x F_x in registers;
//      y-owner (y-line, t): loads its line of q, F_y, D_y F_y -> published
//      x-line-major;  z-owner (z-line, t): likewise for z.
//      (each owner recomputes the pointwise flux it needs from q: cheaper
//      than exchanging flux planes, and A needs no barrier inside)
//   B  x-owner: rate = ((-D_x F_x) - D_y F_y) - D_z F_z (predictor.py:86-90
//      order), written in place over its own partial row;
//   C  node (spatial node, all t): q_new = dt gw.rate + g0 u, residual.
// Three barriers per sweep.  The startup rates and the volume integral use
// the same line ownership on the spatial tile.  Every layout was checked with
// tools/bankcheck.py to be free of bank conflicts at P = 5.
// Residual norms are reduced per element in a fixed order (bitwise
// deterministic); an element freezes at its first converged sweep
// (>= min_iter).  SURVEY.md Appendix A: per-element stopping differs from
// the reference's global rule by <= 1e-14.
#include <algorithm>

#include <cstdlib>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace adg {

#ifndef ADG_PASS_UNROLL
#define ADG_PASS_UNROLL 2
#endif
// dedicated u^n prefetch buffer for 3-D tiles too (0: 1-D / 2-D only, for A/B)
#ifndef ADG_PF_3D
#define ADG_PF_3D 1
#endif
#define ADG_PF_DED3(D) ((D) <= 2 || ADG_PF_3D)
constexpr int kPassUnroll = ADG_PASS_UNROLL;

template <int D, int P>
struct PredCfg {
  static constexpr int M = D + 2;
  static constexpr int PD = ipow(P, D);      // spatial nodes = threads per element
  static constexpr int PT = PD * P;          // space-time nodes
  static constexpr int TILE = PT * M;        // doubles in one space-time tile
  // space-time tile and x-line-major partial rows share padded strides: a
  // node's (or a row's) P x m block is contiguous (LS doubles); 3-D P = 4
  // and P = 6 pad the middle axis by one double (even strides would put
  // every owner role's lanes on a few banks; tools/bankcheck.py)
  static constexpr int LS = P * M;
  // 2-D: node stride LS + 1 and an element stride chosen mod 16 doubles
  // (element tiles of a CTA would otherwise start on the same bank)
  static constexpr int QPAD = (D == 3 && (P == 4 || P == 6)) ? 1 : 0;
  static constexpr int QK = LS + ((D == 2 && P >= 3) ? 1 : 0);
  static constexpr int QJ = P * QK + QPAD;
  static constexpr int QI = P * QJ;
  static constexpr int TILEP = D == 3 ? P * QI : (D == 2 ? P * P * QK : TILE);
  static constexpr int TILE_PAD = TILE + (TILE & 1);
  // 3-D tiles from N=5 up exchange the y and z partials one after the other
  // through a single buffer, so N=5/6 tiles fit two CTAs and N=6 one CTA of
  // shared memory (instead of the L2 slab); N<=4 keeps both in flight
#ifndef ADG_SEQ_YZ_MINP
#define ADG_SEQ_YZ_MINP 6
#endif
  static constexpr bool SEQ_YZ = (D == 3 && P >= ADG_SEQ_YZ_MINP);
  static constexpr int NBUF = D == 3 ? (SEQ_YZ ? 2 : 3) : 2;   // Q + partial buffers
  static constexpr int SPAT = D * PD * M;        // per-direction spatial pieces
  static constexpr int RSZ0 = TILEP > SPAT ? TILEP : SPAT;
#ifndef ADG_TILE_BUDGET_KB
#define ADG_TILE_BUDGET_KB 110
#endif
  static constexpr int BUDGET = ADG_TILE_BUDGET_KB * 1024;  // bytes of tiles per CTA (>= 2 CTAs/SM)
  // elements per CTA by thread count; 3-D tiles from P = ADG_LONE_MINP up
  // run one element per CTA (the lone-element schedule: prefetch, warp
  // residual reduction, direct volume stores)
#ifndef ADG_LONE_MINP
#define ADG_LONE_MINP 3
#endif
  static constexpr int EPB_T = (D == 3 && P >= ADG_LONE_MINP) ? 1 : ((256 / PD) > 0 ? (256 / PD) : 1);
  static constexpr int EPB_S0 = (BUDGET / (NBUF * RSZ0 * 8)) > 0 ? (BUDGET / (NBUF * RSZ0 * 8)) : 1;
  // face-trace staging: the 2D trace blocks of an element are assembled in
  // shared memory behind the published fbar and leave with cp.async.bulk
  // (one 16-byte-aligned bulk store per face) instead of 40-byte-strided
  // per-thread stores
  static constexpr int TB = PD * M + ((PD * M) & 1);
  static constexpr int FBAR = D * PD * M;
  static constexpr int ST_OFF = FBAR + (FBAR & 1);
  // u^n of the CTA's next element is prefetched (cp.async) into the tail of
  // the z-partial buffer, which is dead from the end of the sweeps until the
  // next element's sweeps (the staged traces run from B1 into its head); the
  // startup stages its states there.  Lone 3-D elements with three buffers
  // (C2: N=4); the regions grow by the few doubles the tail needs
#ifndef ADG_PREFETCH_U
#define ADG_PREFETCH_U 1
#endif
  static constexpr bool PREFETCH = ADG_PREFETCH_U && NBUF == 3 && (EPB_T < EPB_S0 ? EPB_T : EPB_S0) == 1;
  static constexpr int PF_NEED = (ST_OFF + 2 * D * TB + PD * M + 1) / 2;
  static constexpr int RSZ1 = (PREFETCH && PF_NEED > RSZ0) ? PF_NEED : RSZ0;
  static constexpr int RSZ = RSZ1 + (RSZ1 & 1);  // region size (even: 16-B aligned)
  static constexpr int EB = D != 2 ? 0 : (P == 3 ? 2 : (P == 5 ? 8 : ((P == 6 || P == 7) ? 2 : 0)));
  static constexpr int ELEM0 = NBUF * RSZ;
  static constexpr int ELEM = D == 2 ? ELEM0 + (((2 * TILEP + EB - ELEM0) % 16) + 16) % 16
                                     : ELEM0;          // doubles per element
  static constexpr int PF_OFF = RSZ - PD * M;    // prefetch slot inside B2
  static constexpr int EPB_S = (BUDGET / (ELEM * 8)) > 0 ? (BUDGET / (ELEM * 8)) : 1;
  static constexpr int EPB = EPB_T < EPB_S ? EPB_T : EPB_S;
  static constexpr int NT = ((EPB * PD + 31) / 32) * 32;
  static constexpr int NW = NT / 32;
  // the residual partials of a lone 3-D element live in its z-partial buffer
  // (dead during the reduction), so the C2 tile (3 x 25 KB) + D/dx fits
  // three CTAs per SM
  // a lone element reduces its residual norms warp by warp (xor shuffles)
  // and every thread folds the NW warp partials itself, in warp order:
  // one barrier per sweep for the residual instead of three
  static constexpr bool WARP_RED = (EPB == 1);
  static constexpr bool RED_IN_TILE = (!WARP_RED && NBUF == 3 && EPB == 1 && 2 * NT <= RSZ);
  static constexpr int RED_DBL = WARP_RED ? 2 * NW : (RED_IN_TILE ? 0 : 2 * NT);
  static constexpr int SMALL_DBL = ((3 * P * P + RED_DBL + 1) / 2) * 2;
  static constexpr int FLAGS = 5 * EPB + 1;
  static constexpr size_t SMALL_BYTES = SMALL_DBL * 8 + ((FLAGS * 4 + 15) / 16) * 16;
  static constexpr size_t TILE_BYTES = (size_t)EPB * ELEM * 8;
  // 1-D / 2-D groups, and the 3-D two-buffer tiles (N = 5, 6), prefetch the
  // next group's u^n into a dedicated buffer behind the tiles (when it still
  // fits the CTAs per SM the tiles allow): at N = 6 the synchronous u^n load
  // held 9 % of the kernel's stall samples (one CTA per SM)
  static constexpr size_t PFB_BYTES = (size_t)EPB * PD * M * 8;
  static constexpr bool SMEM_TILES0 = (SMALL_BYTES + TILE_BYTES) <= 220 * 1024;
  static constexpr int CTAS0 = (int)((228 * 1024) / (SMALL_BYTES + TILE_BYTES + 1024));
  static constexpr bool PF_DED = ADG_PREFETCH_U && !PREFETCH && ADG_PF_DED3(D) && SMEM_TILES0 &&
      (SMALL_BYTES + TILE_BYTES + PFB_BYTES) <= 220 * 1024 &&
      (int)((228 * 1024) / (SMALL_BYTES + TILE_BYTES + PFB_BYTES + 1024)) >= CTAS0;
  static constexpr bool SMEM_TILES = SMEM_TILES0;
  static constexpr size_t SMEM_BYTES =
      SMALL_BYTES + (SMEM_TILES ? TILE_BYTES : 0) + (PF_DED ? PFB_BYTES : 0);
  // resident CTAs per SM the shared footprint allows (228 KB, 1 KB reserved
  // per CTA); passed to __launch_bounds__ so registers do not become the limit
  static constexpr int MINB0 = (int)((228 * 1024) / (SMEM_BYTES + 1024));
  static constexpr int MINB_R = (65536 / (128 * NT)) > 0 ? 65536 / (128 * NT) : 1;  // >= 128 regs
  static constexpr int MINB1 = MINB0 < MINB_R ? MINB0 : MINB_R;
#ifndef ADG_MINB_CAP
#define ADG_MINB_CAP 3
#endif
  // at least 12 warps per SM worth of CTAs before registers may grow past 170
  static constexpr int MINB_CAP = (384 / NT) > ADG_MINB_CAP ? (384 / NT) : ADG_MINB_CAP;
  static constexpr int MINB = MINB1 < 1 ? 1 : (MINB1 > MINB_CAP ? MINB_CAP : MINB1);
  // spatial line tasks (startup / volume): D directions x P^(D-1) lines
  static constexpr int NTASK = D * (PD / P);
  static constexpr bool TR_STAGE = SMEM_TILES && ((NBUF - 1) * RSZ >= ST_OFF + 2 * D * TB);
  static_assert(!PREFETCH || (EPB == 1 && SMEM_TILES && TR_STAGE), "prefetch layout");
};

struct PredArgs {
  const double* u;
  const double* q_init;   // optional starting iterate [E][P^d][P_t][m] (picard_solve initial=)
  const double* dt;
  double* q_out;
  double* vol;
  double* traces;
  uint8_t* pred_bad;
  int32_t* sweeps;
  double* ws;          // global tile workspace (large-tile variant)
  int64_t n_elem;      // elements this launch processes (u, vol, traces offset to the first)
  int64_t tr_elems;    // elements per face plane of the trace arrays (the whole grid)
  double dx[3];
  double gamma;
  double tol;
  int max_iter;
  int min_iter;
  int prim;            // predictor_mode: 0 conservative, 1 primitive
  int startup_only;    // stop after the startup guess (startup_guess): no sweeps,
                       // q_out keeps the iterate variables
  int fold;            // ADG_GRID_FOLD_STATE: vol <- u^n + vol / mass
  // D / dx_dir for the three directions, [dir][P][P] (rows packed with the
  // launch's P).  Kernel parameters live in the constant bank, so every
  // contraction coefficient is a DFMA constant operand: no shared-memory
  // wavefronts for the uniform matrices
  double dd[3 * kMaxP * kMaxP];
};

// spatial node index from per-axis indices (row-major, last axis fastest)
template <int D, int P>
__device__ __forceinline__ int node3(int i, int j, int k) {
  if (D == 3) return (i * P + j) * P + k;
  if (D == 2) return i * P + j;
  return i;
}
// x-line index (== the x-owner's item); y/z partial rows are x-line-major
template <int D, int P>
__device__ __forceinline__ int xline(int j, int k, int t) {
  return D == 3 ? t + P * k + P * P * j : (D == 2 ? t + P * j : t);
}

// offset of spatial node (i, j, k)'s P x m block in the padded tile, and of
// x-line row (j, k, t) in the padded partial buffers
template <int D, int P>
__device__ __forceinline__ int noff(int i, int j, int k) {
  using C = PredCfg<D, P>;
  if (D == 3) return i * C::QI + j * C::QJ + k * C::QK;
  return node3<D, P>(i, j, k) * C::QK;
}
template <int D, int P>
__device__ __forceinline__ int roff(int j, int k, int t) {
  using C = PredCfg<D, P>;
  if (D == 3) return j * C::QI + k * C::QJ + t * C::QK;
  return xline<D, P>(j, k, t) * C::QK;
}

// Contract one direction of a spatial (single time level) field held
// node-major in shared memory: out[node] = sum_l W[row(node)][l] X[line node l].
// Executed as line tasks: task -> (dir, line); the line's P states are loaded,
// transformed pointwise by `pre` (flux of the state, or identity), contracted
// with the P x P matrix W_dir and written node-major into part[dir].
// The direction is a runtime value (strides, flux normal, matrix offset), so
// lanes of different directions run one instruction stream: no divergence
// and one copy of the code per call site.
// Used for the two startup rates (predictor.py:99-126) and the volume
// integral's stiffness contraction (corrector.py:169-176).
template <int D, int P, int MODE>
__device__ __forceinline__ void spatial_line_task(const double* __restrict__ X,
                                                  double* __restrict__ part,
                                                  const double* __restrict__ W, double gm1,
                                                  int dir, int line) {
  // MODE 0: X = states [node][v], pre = flux along dir, W = D/dx (all dirs)
  // MODE 1: X = per-direction rows X[dir][node][v], W = stiffness (shared)
  // MODE 2: X = primitive states [node][v], no pre (gradients), W = D/dx
  using C = PredCfg<D, P>;
  constexpr int M = C::M, PD = C::PD;
  const int ta = D == 3 ? line / P : line;
  const int tb = D == 3 ? line % P : 0;
  // first node and node stride of the line (row-major, last axis fastest)
  int base, stride;
  if (D == 3) {
    base = dir == 0 ? ta * P + tb : (dir == 1 ? ta * P * P + tb : ta * P * P + tb * P);
    stride = dir == 0 ? P * P : (dir == 1 ? P : 1);
  } else if (D == 2) {
    base = dir == 0 ? ta : ta * P;
    stride = dir == 0 ? P : 1;
  } else {
    base = 0;
    stride = 1;
  }
  const double* Xd = MODE == 1 ? X + dir * PD * M : X;
  double x[P][M];
#pragma unroll
  for (int l = 0; l < P; ++l) {
    const int nd = base + l * stride;
    if (MODE == 0) {
      double q[M];
#pragma unroll
      for (int v = 0; v < M; ++v) q[v] = Xd[nd * M + v];
      flux_axis_dyn<D>(q, gm1, dir, x[l]);
    } else {
#pragma unroll
      for (int v = 0; v < M; ++v) x[l][v] = Xd[nd * M + v];
    }
  }
  const double* Wd = MODE != 1 ? W + dir * P * P : W;
  double* pd = part + dir * PD * M;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    double y[M];
#pragma unroll
    for (int v = 0; v < M; ++v) y[v] = 0.0;
#pragma unroll
    for (int l = 0; l < P; ++l) {
      const double d = Wd[i * P + l];
#pragma unroll
      for (int v = 0; v < M; ++v) y[v] = fma(d, x[l][v], y[v]);
    }
    const int nd = base + i * stride;
#pragma unroll
    for (int v = 0; v < M; ++v) pd[nd * M + v] = y[v];
  }
}

// Contract each direction of a spatial (single time level) field held
// node-major in shared memory, as D x P^(D-1) line tasks spread over the
// element's threads; used for the two startup rates (predictor.py:99-126)
// and the volume integral's stiffness contraction (corrector.py:169-176).
template <int D, int P, int MODE>
__device__ __forceinline__ void spatial_line_tasks(const double* __restrict__ X,
                                                   double* __restrict__ part,
                                                   const double* __restrict__ W, double gm1,
                                                   int item) {
  using C = PredCfg<D, P>;
  constexpr int PD = C::PD, PF = PD / P;
  // a lone element whose direction groups fit in whole warps: warp-aligned
  // tasks (dir = tid / WPD): the matrix offset is warp-uniform
  constexpr int WPD = ((PF + 31) / 32) * 32;
  if constexpr (C::EPB == 1 && D * WPD <= C::NT) {
    const int tid = threadIdx.x;
    const int dir = tid / WPD;
    const int line = tid - dir * WPD;
    if (line < PF && dir < D) spatial_line_task<D, P, MODE>(X, part, W, gm1, dir, line);
    return;
  }
  for (int task = item; task < C::NTASK; task += PD) {
    const int dir = task / PF;
    spatial_line_task<D, P, MODE>(X, part, W, gm1, dir, task - dir * PF);
  }
}

// PRIM = 1: predictor_mode="primitive" (predictor.py:94-96, :109-112,
// :165-189): the startup guess and the Picard iterate live in primitive
// variables and the rate is primitive_rhs(v, grad v); gradients travel
// through the same owner passes as the conservative flux derivatives; the
// converged tile is converted back before the admissibility screen.
template <int D, int P, int PRIM>
__global__ void __launch_bounds__(PredCfg<D, P>::NT, PredCfg<D, P>::MINB)
predict_kernel(const __grid_constant__ PredArgs a) {
  using C = PredCfg<D, P>;
  constexpr int M = C::M, PD = C::PD, EPB = C::EPB, NT = C::NT, LS = C::LS;
  constexpr int TP = C::RSZ;
  const DegreeTables& T = tab<P>();
  extern __shared__ __align__(16) double smem[];
  double* Ds = smem;                          // [3][P][P] D / dx_dir
  int* fl = reinterpret_cast<int*>(Ds + 3 * P * P + C::RED_DBL);
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
  // [NT][2] residual partials
  double* red = C::RED_IN_TILE ? tiles + 2 * C::RSZ : Ds + 3 * P * P;

  const int tid = threadIdx.x;
  // padding lanes (tid >= EPB*PD) shadow the last item of the last element:
  // they execute the same instructions on the same data (duplicate stores of
  // identical values are benign), so no branch diverges inside a warp; they
  // only contribute zeros to the residual reduction
  const bool lane_ok = tid < EPB * PD;
  const int el = lane_ok ? tid / PD : EPB - 1;
  const int item = lane_ok ? tid - el * PD : PD - 1;
  const double gm1 = a.gamma - 1.0;
  const double dt = *a.dt;
  const int max_iter = a.max_iter;

  // D / dx per direction: 3-D reads them as uniform constant-bank operands
  // (no shared wavefronts on the bottleneck pipe); 1-D / 2-D stage them in
  // shared memory, where ptxas otherwise hoists the constants into registers
  // and spills
  if constexpr (D < 3) {
    for (int x = tid; x < D * P * P; x += NT) Ds[x] = a.dd[x];
  }
  const double* DD = D == 3 ? a.dd : Ds;
  const double* Dx = DD;
  const double* Dy = DD + P * P;
  const double* Dz = DD + 2 * P * P;

  // role coordinates; item is the owned line / node in every role
  const int ni = (D == 3) ? item / (P * P) : (D == 2 ? item / P : item);
  const int nj = (D == 3) ? (item / P) % P : (D == 2 ? item % P : 0);
  const int nk = (D == 3) ? item % P : 0;
  const int xt = item % P;                                            // x: [j][k][t]
  const int xk = (D == 3) ? (item / P) % P : 0;
  const int xj = (D == 3) ? item / (P * P) : (D == 2 ? item / P : 0);
  const int yi = item % P;                                            // y: [k][t][i]
  const int yt = (D == 3) ? (item / P) % P : item / P;
  const int yk = (D == 3) ? item / (P * P) : 0;
  const int zj = item % P;                                            // z: [t][i][j]
  const int zi = (item / P) % P;
  const int zt = item / (P * P);
  const int qn0 = noff<D, P>(ni, nj, nk);   // node role: own node block in the tile
  const int xr0 = roff<D, P>(xj, xk, xt);   // x-owner: own row in the partial buffers

  // volume-integral scale of this thread's node per direction,
  // (dt |Omega| / dx_j) (w_tensor / w_row) as corrector.py:172-176 forms it;
  // element-independent, so formed once
  double vcoef[D];
  double rmass;   // 1 / (|cell| w_node): ADG_GRID_FOLD_STATE
  {
    const double cv = a.dx[0] * (D >= 2 ? a.dx[1] : 1.0) * (D == 3 ? a.dx[2] : 1.0);
    const double wnode = T.weights[ni] * (D >= 2 ? T.weights[nj] : 1.0) *
                         (D == 3 ? T.weights[nk] : 1.0);
#pragma unroll
    for (int dir = 0; dir < D; ++dir) {
      const int row = dir == 0 ? ni : (dir == 1 ? nj : nk);
      vcoef[dir] = (dt * cv / a.dx[dir]) * (wnode / T.weights[row]);
    }
    rmass = 1.0 / (cv * wnode);
  }
  // a lone element's volume block leaves straight from registers (strided
  // 8-byte stores; L2 merges the sectors) instead of through shared memory
  // and a barrier
#ifndef ADG_VOL_DIRECT
#define ADG_VOL_DIRECT 1
#endif
  constexpr bool VOL_DIRECT = ADG_VOL_DIRECT && EPB == 1;
#ifndef ADG_VOL_NODE
#define ADG_VOL_NODE 0   // (no ADG_GRID_FOLD_STATE in this variant)
#endif
  constexpr bool VOL_NODE = ADG_VOL_NODE && VOL_DIRECT;

  const int64_t ngroups = (a.n_elem + EPB - 1) / EPB;
  // asynchronous copy of element ge's u^n block into dst (PREFETCH layout)
  auto prefetch_u = [&](int64_t ge, double* dst) {
    const double* src = a.u + (size_t)ge * PD * M;
    for (int x = tid; x < PD * M; x += NT) cp_async8(dst + x, src + x);
    cp_async_commit();
  };
  // PF_DED: the whole next group (contiguous elements) into pfb
  double* pfb = C::PF_DED ? tiles + (size_t)EPB * C::ELEM : nullptr;
  auto prefetch_group = [&](int64_t gg) {
    const int64_t e0 = gg * EPB;
    const int64_t ne = (a.n_elem - e0) < EPB ? (a.n_elem - e0) : EPB;
    const double* src = a.u + (size_t)e0 * PD * M;
    for (int x = tid; x < ne * PD * M; x += NT) cp_async8(pfb + x, src + x);
    cp_async_commit();
  };
  if (C::PREFETCH && (int64_t)blockIdx.x < ngroups)
    prefetch_u(blockIdx.x, tiles + 2 * C::RSZ + C::PF_OFF);
  if (C::PF_DED && (int64_t)blockIdx.x < ngroups) prefetch_group(blockIdx.x);
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t e = g * EPB + el;
    const bool valid = e < a.n_elem;
    double* Q = tiles + el * C::ELEM;
    double* B1 = Q + TP;       // y partials / rate (x-line-major); startup+volume scratch
    double* B2 = Q + 2 * TP;   // z partials (D == 3)
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

    // ---------------- startup guess --------------------------------------
    // k = L(w) = ((-D_x F_x) - D_y F_y) - D_z F_z at the spatial nodes,
    // w = u (k1) then u + dt k1 (k2); states staged node-major in Q[:PD*M]
    double* W0 = C::PREFETCH ? B2 + C::PF_OFF
                             : (C::PF_DED ? pfb + el * PD * M : Q);   // staged states [node][v]
    double* PA = B1;                // per-direction pieces [dir][node][v]
    double uu[M];   // u^n (conservative), or its primitive state (PRIM)
    double k1[M];
    double k2[M];
    // u^n of the group's elements: coalesced cooperative copy into each
    // element's W0 (consecutive threads, consecutive doubles), then every
    // node thread takes its own state from shared memory
    if constexpr (C::PREFETCH || C::PF_DED) {
      cp_async_wait_all();   // this thread's part of u^n has landed in W0
    } else {
      for (int x = tid; x < EPB * PD * M; x += NT) {
        const int ee = x / (PD * M);
        const int off = x - ee * (PD * M);
        if (g * EPB + ee < a.n_elem)
          tiles[ee * C::ELEM + off] = a.u[(size_t)(g * EPB + ee) * PD * M + off];
      }
    }
    __syncthreads();
    if (valid) {
#pragma unroll
      for (int v = 0; v < M; ++v) uu[v] = W0[item * M + v];
      if (PRIM) {
        double vv[M];
        cons_to_prim<D>(uu, gm1, vv);
#pragma unroll
        for (int v = 0; v < M; ++v) uu[v] = vv[v];
      }
    }
    if (PRIM) {
      __syncthreads();   // every lane has read its raw state (padding lanes share one)
      if (valid && lane_ok) {
#pragma unroll
        for (int v = 0; v < M; ++v) W0[item * M + v] = uu[v];
      }
    }
    const int npass = a.q_init ? 0 : (P >= 3 ? 2 : 1);
#pragma unroll kPassUnroll
    for (int pass = 0; pass < npass; ++pass) {
      // pass 0 reads the u^n staged before the barrier above (PRIM
      // rewrites it with primitive states first)
      if (pass > 0 || PRIM) __syncthreads();
      if (valid) spatial_line_tasks<D, P, PRIM ? 2 : 0>(W0, PA, DD, gm1, item);
      __syncthreads();
      double* kk = pass == 0 ? k1 : k2;
      if (valid) {
        if (PRIM) {
          double gr[D][M], w[M];   // w: the staged state (u, then u + dt k1)
#pragma unroll
          for (int dir = 0; dir < D; ++dir)
#pragma unroll
            for (int v = 0; v < M; ++v) gr[dir][v] = PA[(dir * PD + item) * M + v];
#pragma unroll
          for (int v = 0; v < M; ++v) w[v] = W0[item * M + v];
          primitive_rhs<D>(w, gr, a.gamma, kk);
        } else {
#pragma unroll
          for (int v = 0; v < M; ++v) {
            double r = 0.0;
#pragma unroll
            for (int dir = 0; dir < D; ++dir) r -= PA[(dir * PD + item) * M + v];
            kk[v] = r;
          }
        }
        if (pass == 0) {
#pragma unroll
          for (int v = 0; v < M; ++v) W0[item * M + v] = uu[v] + dt * k1[v];
        }
      }
    }
    if (!C::PREFETCH && !C::PF_DED) __syncthreads();   // W0 (inside Q) is about to be overwritten
    if (valid && a.q_init) {
      // caller's starting iterate (picard_solve initial=, predictor.py:159-162)
      const double* qi = a.q_init + (size_t)e * C::TILE + (size_t)item * LS;
#pragma unroll
      for (int x = 0; x < LS; ++x) Q[qn0 + x] = qi[x];
    } else if (valid) {
#pragma unroll
      for (int t = 0; t < P; ++t) {
        const double s = T.nodes[t] * dt;
        if (P <= 2) {
#pragma unroll
          for (int v = 0; v < M; ++v) Q[qn0 + t * M + v] = uu[v] + s * k1[v];
        } else {
          const double c2 = 0.5 * s * s / dt;
#pragma unroll
          for (int v = 0; v < M; ++v)
            Q[qn0 + t * M + v] = uu[v] + s * k1[v] + c2 * (k2[v] - k1[v]);
        }
      }
    }
    // the previous group's staged traces must be read out before the sweeps
    // reuse B1 / B2
    if (C::TR_STAGE && tid < EPB) bulk_wait_read_all();
    __syncthreads();

    // ---------------- Picard sweeps -----------------------------------
    int it = 0;
    bool fz = !valid;   // WARP_RED: the lone element's frozen flag, same in every thread
    for (; it < max_iter; ++it) {
      if (C::WARP_RED ? fz : *all_frozen) break;
      const bool work = valid && !(C::WARP_RED ? fz : frozen[el]);
      double rate[P][M];             // conservative: the rate; PRIM: first the x-gradient
      double ql[PRIM ? P : 1][M];    // PRIM: the x-owner's primitive states
      double gyr[(PRIM && C::SEQ_YZ) ? P : 1][M];
      // pointwise pre-transform of a line state: directional flux, or the
      // primitive state itself (gradients)
      auto pre = [&](const double* q, int dir, double* out) {
        if (PRIM) {
#pragma unroll
          for (int v = 0; v < M; ++v) out[v] = q[v];
        } else {
          flux_axis<D>(q, gm1, dir, out);
        }
      };
      // Line contraction, l-outer: each line state is loaded, transformed by
      // `pre` and folded into all P outputs at once (acc[i] += W[i][l] f_l;
      // same per-output fma order as a row-by-row mat-vec, but only one
      // transformed state is live instead of P)
      // (3-D: l-outer; 1-D / 2-D keep the transformed line and contract row
      // by row, which ptxas allocates with fewer spills there; both give
      // each output the same fma order)
      auto line_pass = [&](auto&& qaddr, int dir, const double* W, double sgn,
                           double (&acc)[P][M]) {
        if constexpr (D < 3) {
          double fl[P][M];
#pragma unroll
          for (int l = 0; l < P; ++l) {
            double q[M];
            const double* src = Q + qaddr(l);
#pragma unroll
            for (int v = 0; v < M; ++v) q[v] = src[v];
            pre(q, dir, fl[l]);
            if (PRIM && dir == 0) {
#pragma unroll
              for (int v = 0; v < M; ++v) ql[PRIM ? l : 0][v] = q[v];
            }
          }
#pragma unroll
          for (int i = 0; i < P; ++i) {
            double y[M];
#pragma unroll
            for (int v = 0; v < M; ++v) y[v] = 0.0;
#pragma unroll
            for (int l = 0; l < P; ++l) {
              const double d = sgn * W[i * P + l];
#pragma unroll
              for (int v = 0; v < M; ++v) y[v] = fma(d, fl[l][v], y[v]);
            }
#pragma unroll
            for (int v = 0; v < M; ++v) acc[i][v] = y[v];
          }
          return;
        }
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
          for (int v = 0; v < M; ++v) acc[i][v] = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          double q[M], f[M];
          const double* src = Q + qaddr(l);
#pragma unroll
          for (int v = 0; v < M; ++v) q[v] = src[v];
          pre(q, dir, f);
          if (PRIM && dir == 0) {
#pragma unroll
            for (int v = 0; v < M; ++v) ql[PRIM ? l : 0][v] = q[v];
          }
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const double d = sgn * W[i * P + l];
#pragma unroll
            for (int v = 0; v < M; ++v) acc[i][v] = fma(d, f[v], acc[i][v]);
          }
        }
      };
      // z-owner: own z-line -> D_z partials, x-line-major rows of dst
      auto zpass = [&](double* dst) {
        double acc[P][M];
        line_pass([&](int l) { return noff<D, P>(zi, zj, l) + zt * M; }, 2, Dz, 1.0, acc);
#pragma unroll
        for (int kk = 0; kk < P; ++kk)
#pragma unroll
          for (int v = 0; v < M; ++v) dst[roff<D, P>(zj, kk, zt) + zi * M + v] = acc[kk][v];
      };
      // y-owner: own y-line -> D_y partials, x-line-major rows of dst
      auto ypass = [&](double* dst) {
        double acc[P][M];
        line_pass([&](int l) { return noff<D, P>(yi, l, yk) + yt * M; }, 1, Dy, 1.0, acc);
#pragma unroll
        for (int jj = 0; jj < P; ++jj)
#pragma unroll
          for (int v = 0; v < M; ++v) dst[roff<D, P>(jj, yk, yt) + yi * M + v] = acc[jj][v];
      };
      // A: y/z-owners publish their partials first, then the x-owner's
      // -D_x F_x (PRIM: +D_x v) accumulates straight into `rate`, so only
      // one P x M block is live at a time
      // y-owner, accumulating: dst += D_y F_y (RMW schedule below)
      auto ypass_add = [&](double* dst) {
        double acc[P][M];
        line_pass([&](int l) { return noff<D, P>(yi, l, yk) + yt * M; }, 1, Dy, 1.0, acc);
#pragma unroll
        for (int jj = 0; jj < P; ++jj)
#pragma unroll
          for (int v = 0; v < M; ++v) dst[roff<D, P>(jj, yk, yt) + yi * M + v] += acc[jj][v];
      };
      // Two-buffer 3-D schedule (conservative mode): the z partials go to B1,
      // the y-owners add theirs in place, and the x-owner subtracts the sum
      // from its own -D_x F_x: rate = -D_x F_x - (D_z F_z + D_y F_y).  Same
      // shared traffic as three buffers, one more barrier, 2/3 of the shared
      // footprint and only one P x M block live per phase.
      constexpr bool RMW = C::SEQ_YZ && !PRIM;
#ifndef ADG_DYN_YZ
#define ADG_DYN_YZ 1
#endif
      constexpr bool DYN_YZ = ADG_DYN_YZ && D == 3 && !PRIM && !C::SEQ_YZ;
      if constexpr (RMW) {
        if (work) zpass(B1);
        __syncthreads();
        if (work) ypass_add(B1);
        __syncthreads();
        if (work) {
          line_pass([&](int l) { return noff<D, P>(l, xj, xk) + xt * M; }, 0, Dx, -1.0,
                    rate);
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int v = 0; v < M; ++v) {
              const double r = rate[i][v] - B1[xr0 + i * M + v];
              B1[xr0 + i * M + v] = r;
            }
        }
      } else {
      if (work) {
        if constexpr (DYN_YZ) {
          // z then y owner through one instruction stream (runtime axis):
          // line nodes base + l * nstride at time slot tt; the P outputs land
          // in the x-line-major rows dbase + kk * dstride, slot `slot`
#pragma unroll 1
          for (int dd = 2; dd >= 1; --dd) {
            const bool zz = dd == 2;
            const int nbase = zz ? zi * C::QI + zj * C::QJ : yi * C::QI + yk * C::QK;
            const int nstride = zz ? C::QK : C::QJ;
            const int tt = zz ? zt : yt;
            const int dbase = zz ? zj * C::QI + zt * C::QK : yk * C::QJ + yt * C::QK;
            const int dstride = zz ? C::QJ : C::QI;
            const int slot = zz ? zi : yi;
            double* dst = zz ? B2 : B1;
            const double* W = DD + dd * P * P;
            double acc[P][M];
#pragma unroll
            for (int i = 0; i < P; ++i)
#pragma unroll
              for (int v = 0; v < M; ++v) acc[i][v] = 0.0;
#pragma unroll
            for (int l = 0; l < P; ++l) {
              double q[M], f[M];
              const double* src = Q + nbase + l * nstride + tt * M;
#pragma unroll
              for (int v = 0; v < M; ++v) q[v] = src[v];
              flux_axis_dyn<D>(q, gm1, dd, f);
#pragma unroll
              for (int i = 0; i < P; ++i) {
                const double d = W[i * P + l];
#pragma unroll
                for (int v = 0; v < M; ++v) acc[i][v] = fma(d, f[v], acc[i][v]);
              }
            }
#pragma unroll
            for (int kk = 0; kk < P; ++kk)
#pragma unroll
              for (int v = 0; v < M; ++v) dst[dbase + kk * dstride + slot * M + v] = acc[kk][v];
          }
        } else {
          if (D == 3 && !C::SEQ_YZ) zpass(B2);
          if (D >= 2) ypass(B1);
        }
        line_pass([&](int l) { return noff<D, P>(l, xj, xk) + xt * M; }, 0, Dx,
                  PRIM ? 1.0 : -1.0, rate);
      }
      if (D >= 2) __syncthreads();
      if (C::SEQ_YZ) {
        // y partials consumed, then the z partials take the same buffer
        if (work) {
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int v = 0; v < M; ++v) {
              if (PRIM) gyr[PRIM ? i : 0][v] = B1[xr0 + i * M + v];
              else rate[i][v] -= B1[xr0 + i * M + v];
            }
        }
        __syncthreads();
        if (work) zpass(B1);
        __syncthreads();
      }
      if (PRIM && work) {
        // rate = primitive_rhs(v, (grad_x, grad_y, grad_z)) at the x-line's nodes
        const double* PZ = C::SEQ_YZ ? B1 : B2;
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double gr[D][M];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            gr[0][v] = rate[i][v];
            if (D >= 2) gr[D >= 2 ? 1 : 0][v] = C::SEQ_YZ ? gyr[(PRIM && C::SEQ_YZ) ? i : 0][v]
                                                           : B1[xr0 + i * M + v];
            if (D == 3) gr[D == 3 ? 2 : 0][v] = PZ[xr0 + i * M + v];
          }
          primitive_rhs<D>(ql[PRIM ? i : 0], gr, a.gamma, rate[i]);
        }
      }
      // B: x-owner completes its rate in place (x-line-major rows of B1)
      if (work) {
        if (!PRIM && D >= 2 && !C::SEQ_YZ) {
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int v = 0; v < M; ++v) rate[i][v] -= B1[xr0 + i * M + v];
        }
        if (!PRIM && D == 3) {
          const double* PZ = C::SEQ_YZ ? B1 : B2;
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int v = 0; v < M; ++v) rate[i][v] -= PZ[xr0 + i * M + v];
        }
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
          for (int v = 0; v < M; ++v) B1[xr0 + i * M + v] = rate[i][v];
      }
      }
      __syncthreads();
      // C: node role, time operator + residual; rate(node, s) sits in the
      // x-line-major row of (nj, nk, s) at slot ni
      double sd = 0.0, sq = 0.0;
      if (work) {
        double r[P][M];
#pragma unroll
        for (int s = 0; s < P; ++s)
#pragma unroll
          for (int v = 0; v < M; ++v) r[s][v] = B1[roff<D, P>(nj, nk, s) + ni * M + v];
#pragma unroll
        for (int t = 0; t < P; ++t) {
          const double g0 = T.g0[t];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            double c = 0.0;
#pragma unroll
            for (int s = 0; s < P; ++s) c = fma(T.gw[t * P + s], r[s][v], c);
            const double qn = c * dt + g0 * uu[v];
            const double dq = Q[qn0 + t * M + v] - qn;
            sd = fma(dq, dq, sd);
            sq = fma(qn, qn, sq);
            Q[qn0 + t * M + v] = qn;
          }
        }
      }
      if constexpr (C::WARP_RED) {
        const int warp = tid >> 5, lane = tid & 31;
        double s1 = lane_ok ? sd : 0.0, s2 = lane_ok ? sq : 0.0;
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
        if (!fz) {
          double t1 = 0.0, t2 = 0.0;
#pragma unroll
          for (int w = 0; w < C::NW; ++w) {
            t1 += red[2 * w];
            t2 += red[2 * w + 1];
          }
          const double res = T.k1_opnorm * sqrt(t1);
          const double scale = 1.0 + sqrt(t2);
          const int c = res <= a.tol * scale;
          if (c && it + 1 >= a.min_iter) fz = true;
          if (tid == 0) {
            conv[0] = c;
            nsw[0] = it + 1;
          }
        }
        // red is rewritten only after the next sweep's two barriers
        continue;
      }
      red[2 * tid] = lane_ok ? sd : 0.0;
      red[2 * tid + 1] = lane_ok ? sq : 0.0;
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

    // B2 is dead until the next element's sweeps: start fetching its u^n
    if (C::PREFETCH && g + gridDim.x < ngroups) prefetch_u(g + gridDim.x, B2 + C::PF_OFF);
    // every lane of the group has passed its startup (pfb is dead) since the
    // sweep loop's barriers
    if (C::PF_DED && g + gridDim.x < ngroups) prefetch_group(g + gridDim.x);
    if (PRIM && !a.startup_only) {
      // q_cons = prim_to_cons(q) (predictor.py:188), each node thread its own
      if (valid) {
#pragma unroll
        for (int t = 0; t < P; ++t) {
          double v[M], q[M];
#pragma unroll
          for (int w = 0; w < M; ++w) v[w] = Q[qn0 + t * M + w];
          prim_to_cons<D>(v, gm1, q);
#pragma unroll
          for (int w = 0; w < M; ++w) Q[qn0 + t * M + w] = q[w];
        }
      }
      __syncthreads();
    }
    // ---------------- admissibility, traces, volume flux sums ----------
    double fb[D][M];   // fbar_dir = sum_t w_t F_dir(q_t) (corrector.py:171)
    if (valid) {
      bool ok = true;
#pragma unroll
      for (int dir = 0; dir < D; ++dir)
#pragma unroll
        for (int v = 0; v < M; ++v) fb[dir][v] = 0.0;
#pragma unroll
      for (int t = 0; t < P; ++t) {
        double q[M];
#pragma unroll
        for (int v = 0; v < M; ++v) q[v] = Q[qn0 + t * M + v];
        double f[D][M];
        ok = flux_all_adm<D>(q, gm1, f) && ok;
        const double wt = T.weights[t];
#pragma unroll
        for (int dir = 0; dir < D; ++dir)
#pragma unroll
          for (int v = 0; v < M; ++v) fb[dir][v] = fma(wt, f[dir][v], fb[dir][v]);
      }
      if (!ok) okf[el] = 0;
      // traces: each owner role writes its own line's face states at block
      // offset item*m (x: [j][k][t], y: [k][t][i], z: [t][i][j])
      // element trace blocks padded to a 16-byte multiple (TMA in the face kernel)
      constexpr int TB = C::TB;
      const size_t face_stride = (size_t)a.tr_elems * TB;
      const size_t eoff = (size_t)e * TB + (size_t)item * M;
      double* stage = B1 + C::ST_OFF;
#pragma unroll
      for (int dir = 0; dir < D; ++dir) {
        double lo[M], hi[M];
#pragma unroll
        for (int v = 0; v < M; ++v) lo[v] = hi[v] = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          const int q0 = dir == 0 ? noff<D, P>(l, xj, xk) + xt * M
                                  : (dir == 1 ? noff<D, P>(yi, l, yk) + yt * M
                                              : noff<D, P>(zi, zj, l) + zt * M);
          const double pl = T.left[l], pr = T.right[l];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            const double qv = Q[q0 + v];
            lo[v] = fma(pl, qv, lo[v]);
            hi[v] = fma(pr, qv, hi[v]);
          }
        }
        if (C::TR_STAGE) {
          double* slo = stage + (2 * dir) * TB + item * M;
#pragma unroll
          for (int v = 0; v < M; ++v) {
            slo[v] = lo[v];
            slo[TB + v] = hi[v];
          }
        } else {
          double* tlo = a.traces + (size_t)(2 * dir) * face_stride + eoff;
          double* thi = tlo + face_stride;
#pragma unroll
          for (int v = 0; v < M; ++v) {
            tlo[v] = lo[v];
            thi[v] = hi[v];
          }
        }
      }
      if (C::TR_STAGE) fence_proxy_async_smem();   // staged traces -> async proxy
      if (a.q_out) {
        double* qo = a.q_out + (size_t)e * C::TILE + (size_t)item * LS;   // unpadded
#pragma unroll
        for (int x = 0; x < LS; ++x) qo[x] = Q[qn0 + x];
      }
      // publish fbar node-major for the stiffness line tasks
#pragma unroll
      for (int dir = 0; dir < D; ++dir)
#pragma unroll
        for (int v = 0; v < M; ++v) B1[(dir * PD + item) * M + v] = fb[dir][v];
    }
    __syncthreads();
    if (C::TR_STAGE && tid < EPB && valid_e[tid]) {
      const size_t face_stride = (size_t)a.tr_elems * C::TB;
      const double* st = tiles + tid * C::ELEM + TP + C::ST_OFF;
      double* dst = a.traces + (size_t)(g * EPB + tid) * C::TB;
#pragma unroll
      for (int f = 0; f < 2 * D; ++f)
        bulk_s2g(dst + (size_t)f * face_stride, st + f * C::TB, C::TB * 8);
      bulk_commit();
    }
    // volume: contrib_dir = stiff x_dir fbar_dir (corrector.py:172-174)
    if constexpr (VOL_NODE) {
      // node form: each node thread contracts the D fbar lines through it
      // (same per-output fma order as the line tasks), scales and stores
      if (valid && lane_ok) {
        double acc[M];
#pragma unroll
        for (int v = 0; v < M; ++v) acc[v] = 0.0;
#pragma unroll
        for (int dir = 0; dir < D; ++dir) {
          const int row = dir == 0 ? ni : (dir == 1 ? nj : nk);
          const int stride = D == 3 ? (dir == 0 ? P * P : (dir == 1 ? P : 1))
                                    : (D == 2 ? (dir == 0 ? P : 1) : 1);
          const double* fl = B1 + (dir * PD + item - row * stride) * M;
          double y[M];
#pragma unroll
          for (int v = 0; v < M; ++v) y[v] = 0.0;
#pragma unroll
          for (int l = 0; l < P; ++l) {
            const double d = T.stiff[row * P + l];
#pragma unroll
            for (int v = 0; v < M; ++v) y[v] = fma(d, fl[l * stride * M + v], y[v]);
          }
#pragma unroll
          for (int v = 0; v < M; ++v) acc[v] += vcoef[dir] * y[v];
        }
        double* vo = a.vol + ((size_t)e * PD + item) * M;
#pragma unroll
        for (int v = 0; v < M; ++v) vo[v] = acc[v];
      }
    } else {
    if (valid) spatial_line_tasks<D, P, 1>(B1, Q, T.stiff, gm1, item);
    __syncthreads();
    if (valid) {
      const double* CB = Q;
      double acc[M];
#pragma unroll
      for (int v = 0; v < M; ++v) acc[v] = 0.0;
#pragma unroll
      for (int dir = 0; dir < D; ++dir) {
#pragma unroll
        for (int v = 0; v < M; ++v) acc[v] += vcoef[dir] * CB[(dir * PD + item) * M + v];
      }
      if (!PRIM && a.fold) {   // w = u^n + vol / mass (uu is the conservative u^n here)
#pragma unroll
        for (int v = 0; v < M; ++v) acc[v] = fma(acc[v], rmass, uu[v]);
      }
      if constexpr (VOL_DIRECT) {
        if (lane_ok) {
          double* vo = a.vol + ((size_t)e * PD + item) * M;
#pragma unroll
          for (int v = 0; v < M; ++v) vo[v] = acc[v];
        }
      } else if (lane_ok) {
        // own row of the dir-0 block is no longer read by anyone: stage there
#pragma unroll
        for (int v = 0; v < M; ++v) Q[item * M + v] = acc[v];
      }
    }
    if constexpr (!VOL_DIRECT) {
      __syncthreads();
      // coalesced copy of the group's volume blocks to HBM
      for (int x = tid; x < EPB * PD * M; x += NT) {
        const int ee = x / (PD * M);
        const int off = x - ee * (PD * M);
        if (g * EPB + ee < a.n_elem)
          a.vol[(size_t)(g * EPB + ee) * PD * M + off] = tiles[ee * C::ELEM + off];
      }
    }
    }
    if (tid < EPB && valid_e[tid]) {
      const int64_t ee = g * EPB + tid;
      a.pred_bad[ee] = (conv[tid] ? 0 : ADG_PRED_NOT_CONVERGED) | (okf[tid] ? 0 : ADG_PRED_INADMISSIBLE);
      a.sweeps[ee] = nsw[tid] ? nsw[tid] : it;
    }
  }
  if (C::TR_STAGE && tid < EPB) bulk_wait_all();
}

template <int D, int P>
static int launch_predict(const PredArgs& a0, cudaStream_t st, int num_sms, double* ws_pool,
                          size_t ws_bytes, std::string* err) {
  using C = PredCfg<D, P>;
  auto kern = a0.prim ? predict_kernel<D, P, 1> : predict_kernel<D, P, 0>;
  static PerDevice attr_set[2];
  if (attr_set[a0.prim ? 1 : 0].first()) {
    if (C::SMEM_BYTES > 48 * 1024) {
      cudaError_t ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)C::SMEM_BYTES);
      if (ce != cudaSuccess) {
        *err = cudaGetErrorString(ce);
        return ADG_ERR_CUDA;
      }
    }
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

size_t predict_workspace_bytes(int dim, int P, int num_sms, int64_t n_elem) {
  if (dim == 1) { ADG_DISPATCH_P(1, ws_need, num_sms) }
  if (dim == 2) { ADG_DISPATCH_P(2, ws_need, num_sms) }
  if (dim == 3) {
    // 3-D P >= 8: the slice-streaming kernel's scratch or the large-tile
    // variant's (primitive mode), whichever is larger
    const size_t s = predict_stream_workspace_bytes(P, num_sms);
    size_t t = 0;
    switch (P) {
      case 8: t = ws_need<3, 8>(num_sms); break;
      case 9: t = ws_need<3, 9>(num_sms); break;
      case 10: t = ws_need<3, 10>(num_sms); break;
      default: { ADG_DISPATCH_P(3, ws_need, num_sms) }
    }
    const size_t ph = (P >= 8 && n_elem > 0) ? predict_phased_workspace_bytes(P, n_elem) : 0;
    const size_t st = s > t ? s : t;
    return st > ph ? st : ph;
  }
  return 0;
}

bool predict_range_supported(const adg_grid* g) { return !predict_stream_supported(g); }

// ADG_GRID_FOLD_STATE: Euler, conservative iterate, shared-tile kernel
bool predict_fold_supported(const adg_grid* g) {
  return g->system == ADG_SYS_EULER && g->mode == ADG_MODE_CONSERVATIVE &&
         !predict_stream_supported(g) && !ADG_VOL_NODE;
}

int predict(const adg_grid* g, const double* u, const double* dt_dev, double tol, int max_iter,
            int min_iter, double* q_out, double* vol, double* traces, uint8_t* pred_bad,
            int32_t* sweeps, cudaStream_t st, int num_sms, double* ws, size_t ws_bytes,
            std::string* err, int64_t e_begin, int64_t e_count, const double* q_init,
            int startup_only) {
  const int64_t n_all =
      g->cells[0] * (g->dim >= 2 ? g->cells[1] : 1) * (g->dim == 3 ? g->cells[2] : 1);
  if (e_count < 0) e_count = n_all - e_begin;
  if (e_begin < 0 || e_begin + e_count > n_all) {
    *err = "element range outside the grid";
    return ADG_ERR_INVALID;
  }
  const bool whole = e_begin == 0 && e_count == n_all;
  if (!whole && !predict_range_supported(g)) {
    *err = "element ranges need the shared-tile predictor (not the 3-D N>=7 phased / stream kernels)";
    return ADG_ERR_UNSUPPORTED;
  }
  // a caller's starting iterate or a startup-only call runs the shared-tile
  // kernel (its large-tile variant for 3-D N >= 7)
  // ADG_PREDICTOR=tile: the shared-tile kernel's large-tile variant for the
  // 3-D N >= 7 grids too (A/B runs against the slice-streaming kernel)
  const char* pv = getenv("ADG_PREDICTOR");
  const bool plain = q_init == nullptr && !startup_only && !(pv && pv[0] == 't');
  const bool fold = (g->flags & ADG_GRID_FOLD_STATE) != 0;
  if (fold && (!predict_fold_supported(g) || startup_only)) {
    *err = "ADG_GRID_FOLD_STATE: not supported for this grid (adg_fold_supported)";
    return ADG_ERR_UNSUPPORTED;
  }
  // 3-D tiles beyond one SM's shared memory (N >= 7): from N = 8 up as phase
  // kernels over element batches with the iterate in HBM
  // (adg_predictor_phased.cu: 30.1 vs 51.4 ms at N = 8, 56.1 vs 78.3 ms at N = 9
  // on 32^3 elements), at N = 7 as one CTA per element streaming time slices
  // through shared memory (adg_predictor_stream.cu: 17.4 vs 18.2 ms);
  // ADG_PREDICTOR=phased / stream forces one of them for A/B runs
  if (plain && predict_phased_supported(g) && !(pv && pv[0] == 's') &&
      (g->degree >= 8 || (pv && pv[0] == 'p')))
    return predict_phased(g, u, dt_dev, tol, max_iter, min_iter, q_out, vol, traces, pred_bad,
                          sweeps, st, num_sms, ws, ws_bytes, err);
  if (plain && predict_stream_supported(g))
    return predict_stream(g, u, dt_dev, tol, max_iter, min_iter, q_out, vol, traces, pred_bad,
                          sweeps, st, num_sms, ws, ws_bytes, err);
  // an element range [e_begin, e_begin + e_count) is the same launch on
  // pointers advanced to its first element; only the trace planes keep the
  // whole grid's stride (the slab decomposition predicts its boundary layers
  // first and overlaps their halo exchange with the interior, decomp.py)
  const int Pn = g->degree + 1;
  int64_t pd = 1;
  for (int j = 0; j < g->dim; ++j) pd *= Pn;
  const int64_t blk = pd * (g->dim + 2);
  const int64_t tb = blk + (blk & 1);
  PredArgs a{};
  a.u = u + e_begin * blk;
  a.q_init = q_init ? q_init + e_begin * blk * Pn : nullptr;
  a.startup_only = startup_only ? 1 : 0;
  a.dt = dt_dev;
  a.q_out = q_out ? q_out + e_begin * blk * Pn : nullptr;
  a.vol = vol + e_begin * blk;
  a.traces = traces + e_begin * tb;
  a.pred_bad = pred_bad + e_begin;
  a.sweeps = sweeps + e_begin;
  a.ws = nullptr;
  a.n_elem = e_count;
  a.tr_elems = n_all;
  if (e_count == 0) return ADG_OK;
  for (int j = 0; j < 3; ++j) a.dx[j] = j < g->dim ? g->dx[j] : 1.0;
  a.gamma = g->gamma;
  a.tol = tol;
  a.max_iter = startup_only ? 0 : (max_iter > 0 ? max_iter : 2 * g->degree + 2);
  a.min_iter = min_iter;
  a.prim = g->mode == ADG_MODE_PRIMITIVE ? 1 : 0;
  a.fold = fold ? 1 : 0;
  {
    // D / dx exactly as the reference forms it (diff / spacing, one IEEE
    // division per entry, basis.py diff; predictor.py:65-71)
    const int Pl = g->degree + 1;
    for (int dir = 0; dir < 3; ++dir)
      for (int x = 0; x < Pl * Pl; ++x)
        a.dd[dir * Pl * Pl + x] = dir < g->dim ? h_tab[g->degree].diff[x] / g->dx[dir] : 0.0;
  }
  const int P = g->degree + 1;
  if (g->dim == 1) { ADG_DISPATCH_P(1, launch_predict, a, st, num_sms, ws, ws_bytes, err) }
  if (g->dim == 2) { ADG_DISPATCH_P(2, launch_predict, a, st, num_sms, ws, ws_bytes, err) }
  if (g->dim == 3) { ADG_DISPATCH_P(3, launch_predict, a, st, num_sms, ws, ws_bytes, err) }
  *err = "unsupported dim/degree";
  return ADG_ERR_UNSUPPORTED;
}

}  // namespace adg
