// adg_predictor_cluster.cu -- the fused ADER-DG predictor for the large 3-D
// space-time tiles (P = N+1 = 8..10: 160-391 KB per element, more than one
// SM's shared memory), as a thread-block cluster.
//
// Same algorithm and outputs as predict_kernel (adg_predictor.cu): startup
// guess (predictor.py:99-126), Picard sweeps with per-element freezing
// (predictor.py:135-191), admissibility (:188-189), face traces (:218-230)
// and the volume integral (corrector.py:141-177).  Layout: a cluster of
// C = P CTAs holds one element; CTA c owns time slice t = c of the tile in
// its shared memory (P^3 x m doubles).  Every spatial operation is
// slice-local; the time operator couples the slices and runs over DSMEM:
// CTA c owns the spatial nodes of x-plane i = c at all times, gathers their
// rates from the P slices (ld.shared::cluster) and scatters the new iterate
// back (st.shared::cluster).  Residual norms and the admissibility verdict are
// combined in a fixed CTA order, so every CTA takes the same decision and
// reruns are bitwise identical.
//
// Threads: 3 P^2 line owners per CTA (x-, y-, z-lines of the slice) run the
// flux + derivative contraction of their line through one runtime-axis code
// path; the x-owner completes the rate of its line from the y/z partials.
#include <cooperative_groups.h>

#include <algorithm>

#include "adg_common.cuh"
#include "adg_internal.h"

namespace cg = cooperative_groups;

namespace adg {

template <int P>
struct ClCfg {
  static constexpr int M = 5;
  static constexpr int C = P;                         // CTAs per cluster (one slice each)
  static constexpr int PP = P * P;
  static constexpr int PD = P * P * P;
  // padded slice layouts (tools/cluster_bankcheck.py: fewest shared-memory
  // wavefronts over the owners' line loads, partial stores and row reads):
  // Q node-major [i][j][k][v] strides (SI, SJ, M); B x-line-major
  // [j][k][i][v] strides (TJ, TK, M)
  static constexpr int SJ = P * M + (P == 8 ? 1 : (P == 10 ? 3 : 0));
  static constexpr int SI = P * SJ;
  static constexpr int TK = P * M + (P == 8 ? 2 : (P == 10 ? 1 : 0));
  static constexpr int TJ = P * TK + (P == 8 ? 1 : 0);
  static constexpr int QSZ = P * SI;
  static constexpr int BSZ = P * TJ;
  static constexpr int QSZP = QSZ + (QSZ & 1);        // 16-byte aligned buffers
  static constexpr int BSZP = BSZ + (BSZ & 1);
  static constexpr int NT = ((3 * PP + 31) / 32) * 32;
  static constexpr int NW = NT / 32;
  // red[NW][2] warp partials, credg[C][2] gathered residual partials,
  // okg[C] gathered verdicts, 4 mbarriers
  static constexpr int SMALL = 2 * NW + 2 * C + C + 4;
  static constexpr size_t SMEM = ((size_t)QSZP + 4 * (size_t)BSZP + ((SMALL + 1) / 2) * 2) * 8;
  static constexpr int MINB = (228 * 1024) / (SMEM + 1024) >= 2 ? 2 : 1;  // CTAs per SM
  static constexpr int TB = PD * M + ((PD * M) & 1);  // trace block (face kernel layout)
};

struct ClArgs {
  const double* u;
  const double* dt;
  double* q_out;
  double* vol;
  double* traces;
  uint8_t* pred_bad;
  int32_t* sweeps;
  int64_t n_elem;
  double dx[3];
  double gamma;
  double tol;
  int max_iter;
  int min_iter;
  double dd[3 * kMaxP * kMaxP];   // D / dx_dir, [dir][P][P] (kernel-parameter constant bank)
};

template <int P>
__global__ void __launch_bounds__(ClCfg<P>::NT, ClCfg<P>::MINB)
predict_cluster_kernel(const __grid_constant__ ClArgs a) {
  using C = ClCfg<P>;
  constexpr int M = C::M, PP = C::PP, PD = C::PD, NT = C::NT, NW = C::NW;
  constexpr int SI = C::SI, SJ = C::SJ, TJ = C::TJ, TK = C::TK;
  const DegreeTables& T = tab<P>();
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double smem[];
  double* Q = smem;                 // slice tile, node-major (padded)
  double* B1 = Q + C::QSZP;         // y partials, then the rate (x-line-major, padded)
  double* B2 = B1 + C::BSZP;        // z partials (x-line-major)
  double* B3 = B2 + C::BSZP;        // k1 (startup), node role's previous iterate (sweeps),
                                    // volume part (final); x-line-major rows
  double* G = B3 + C::BSZP;         // gathered from the cluster (x-line-major rows, slot
                                    // = source slice): rates (sweeps), volume parts (final)
  double* red = G + C::BSZP;        // [NW][2] warp partials
  double* credg = red + 2 * NW;     // [C][2] residual partials of every slice
  double* okg = credg + 2 * C::C;   // [C] admissibility verdict of every slice
  uint64_t* bars = reinterpret_cast<uint64_t*>(okg + C::C);
  uint64_t* barG = bars;            // G complete (st.async complete_tx)
  uint64_t* barQ = bars + 1;        // this slice's new iterate complete
  uint64_t* barC = bars + 2;        // credg complete
  uint64_t* barF = bars + 3;        // okg complete (its own barrier: a fast CTA's verdict
                                    // must not count toward a residual phase still open)

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int c = (int)cluster.block_rank();       // time slice of this CTA
  const int64_t cid = blockIdx.x / C::C;
  const int64_t ncl = gridDim.x / C::C;
  const double gm1 = a.gamma - 1.0;
  const double dt = *a.dt;
  const double tn = T.nodes[c];
  const double wtc = T.weights[c];

  // line ownership: role 0/1/2 = x/y/z line (a0, b0) of the slice; role 3: idle
  const int role = tid / PP;
  const int rr = tid - role * PP;
  const int a0 = rr / P, b0 = rr - (rr / P) * P;
  const bool owner = role < 3;
  const int dir = owner ? role : 0;
  // line nodes: Q + qbase + l * qstride; node index (unpadded) nbase + l * nstride
  const int qbase = role == 0 ? a0 * SJ + b0 * M : (role == 1 ? a0 * SI + b0 * M : a0 * SI + b0 * SJ);
  const int qstride = role == 0 ? SI : (role == 1 ? SJ : M);
  const int nbase = role == 0 ? a0 * P + b0 : (role == 1 ? a0 * PP + b0 : a0 * PP + b0 * P);
  const int nstride = role == 0 ? PP : (role == 1 ? P : 1);
  // y/z partials -> x-line-major rows: y (i=a0, k=b0) output j: B(j, b0, a0);
  // z (i=a0, j=b0) output k: B(b0, k, a0)
  const int pbase = role == 1 ? b0 * TK + a0 * M : b0 * TJ + a0 * M;
  const int pstride = role == 1 ? TJ : TK;
  double* pdst = role == 1 ? B1 : B2;
  const double* Wd = a.dd + dir * PP;
  // x-owner row: x-line (j, k) = (a0, b0); node role: node (c, a0, b0)
  const int xrow = a0 * TJ + b0 * TK;
  const bool node_role = tid < PP;
  constexpr int TPR = (P + 2) / 3;                // times per owner in the time operator
  const int tlo = role * TPR, thi = tlo + TPR < P ? tlo + TPR : P;
  const int nnode = c * PP + rr;                 // valid when node_role (unpadded index)
  const int qnode = c * SI + a0 * SJ + b0 * M;   // its padded offset in Q

  // volume scales (dt |Omega| / dx_dir) (corrector.py:172-176)
  const double cv = a.dx[0] * a.dx[1] * a.dx[2];
  const double sc0 = dt * cv / a.dx[0], sc1 = dt * cv / a.dx[1], sc2 = dt * cv / a.dx[2];

  // one line's P states -> pointwise transform -> P x P contraction, l-outer
  // (mode 0: flux along dir with D/dx; mode 1: with the stiffness, plus the
  // admissibility screen)
  auto line_contract = [&](int mode, double (&acc)[P][M], bool& ok) {
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int v = 0; v < M; ++v) acc[i][v] = 0.0;
#pragma unroll
    for (int l = 0; l < P; ++l) {
      double q[M], f[M];
      const double* src = Q + qbase + l * qstride;
#pragma unroll
      for (int v = 0; v < M; ++v) q[v] = src[v];
      flux_axis_dyn<3>(q, gm1, dir, f);
      if (mode == 1) ok = ok && admissible<3>(q, gm1);
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const double d = mode == 0 ? Wd[i * P + l] : T.stiff[i * P + l];
#pragma unroll
        for (int v = 0; v < M; ++v) acc[i][v] = fma(d, f[v], acc[i][v]);
      }
    }
  };
  auto publish = [&](const double (&acc)[P][M]) {
#pragma unroll
    for (int o = 0; o < P; ++o)
#pragma unroll
      for (int v = 0; v < M; ++v) pdst[pbase + o * pstride + v] = acc[o][v];
  };
  // u^n of element ee into the padded Q (asynchronous 8-byte copies)
  auto fetch_u = [&](int64_t ee) {
    const double* ue = a.u + (size_t)ee * PD * M;
    for (int x = tid; x < PD * M; x += NT) {
      const int n = x / M, v = x - (x / M) * M;
      const int i = n / PP, j = (n / P) % P, k = n % P;
      cp_async8(Q + i * SI + j * SJ + k * M + v, ue + x);
    }
    cp_async_commit();
  };

  // DSMEM pushes: st.async to the consumer CTA's buffer, completing bytes on
  // its mbarrier (no cluster-wide barrier or fence per exchange)
  auto push = [&](double* local_dst, int rank, uint64_t* local_bar, double v) {
    uint32_t ra, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local_dst)), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(local_bar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];"
                 ::"r"(ra), "d"(v), "r"(rb) : "memory");
  };
  auto wait = [&](uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
          " selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
  };
  // cluster barrier without the release/acquire fences (MEMBAR.GPU + L1
  // invalidation in SASS): every cross-CTA datum travels by st.async with
  // mbarrier completion; these barriers only order buffer reuse (reads whose
  // values were already consumed) and the mbarrier initialisation (published
  // by fence.mbarrier_init)
  auto cluster_barrier = [&]() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n barrier.cluster.wait.aligned;" ::: "memory");
  };
  uint32_t phG = 0, phQ = 0, phC = 0, phF = 0;   // parity of each barrier's current phase
  if (tid == 0) {
    mbar_init(barG, 1);
    mbar_init(barQ, 1);
    mbar_init(barC, 1);
    mbar_init(barF, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_barrier();   // barriers initialised cluster-wide before any push

  if (cid < a.n_elem) fetch_u(cid);
  for (int64_t e = cid; e < a.n_elem; e += ncl) {
    cluster_barrier();   // every CTA of the cluster is done with the previous element
    // ---------------- startup guess (each CTA for its own slice) ----------
    const double* ue = a.u + (size_t)e * PD * M;
    double uu[M];     // u^n at node (c, a0, b0) (every owner shares the time operator)
    if (owner) {
#pragma unroll
      for (int v = 0; v < M; ++v) uu[v] = ue[nnode * M + v];
    }
    cp_async_wait_all();
    __syncthreads();
    double kc[M];     // x-owner: k2 at node (c, a0, b0)
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      double acc[P][M];
      bool dummy = true;
      if (owner) line_contract(0, acc, dummy);
      if (role == 1 || role == 2) publish(acc);
      __syncthreads();
      if (role == 0) {
        // k = ((-D_x F_x) - D_y F_y) - D_z F_z at the x-line's nodes
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double* qn = Q + qbase + i * qstride;
#pragma unroll
          for (int v = 0; v < M; ++v) {
            const double k = (-acc[i][v] - B1[xrow + i * M + v]) - B2[xrow + i * M + v];
            if (pass == 0) {
              B3[xrow + i * M + v] = k;                 // k1
              qn[v] = qn[v] + dt * k;                   // w = u + dt k1
            } else {
              const double s = tn * dt;
              const double c2 = 0.5 * s * s / dt;
              const double k1 = B3[xrow + i * M + v];
              qn[v] = ue[(nbase + i * nstride) * M + v] + s * k1 + c2 * (k - k1);
              if (i == c) kc[v] = k;
            }
          }
        }
        if (pass == 1) {
          // the same thread is the node role of node (c, a0, b0): its
          // startup iterate at every time (bitwise what CTA t forms for its
          // slice) goes to its own B3 row, slot t -- the node role reads the
          // previous iterate there instead of over DSMEM
          double k1c[M];
#pragma unroll
          for (int v = 0; v < M; ++v) k1c[v] = B3[xrow + c * M + v];
#pragma unroll
          for (int t = 0; t < P; ++t) {
            const double s = T.nodes[t] * dt;
            const double c2 = 0.5 * s * s / dt;
#pragma unroll
            for (int v = 0; v < M; ++v) B3[xrow + t * M + v] = uu[v] + s * k1c[v] + c2 * (kc[v] - k1c[v]);
          }
        }
      }
      __syncthreads();
    }

    // ---------------- Picard sweeps -----------------------------------
    int it = 0, conv = 0, nsw = 0;
    bool fz = false;
    for (; it < a.max_iter && !fz; ++it) {
      if (tid == 0) {
        // arm this sweep's phases: all P^3 m rates of x-plane c, the slice's
        // new iterate, the C residual pairs (pushes may already be landing)
        mbar_expect_tx(barG, PD * M * 8);
        mbar_expect_tx(barQ, PD * M * 8);
        mbar_expect_tx(barC, C::C * 16);
      }
      double acc[P][M];
      bool dummy = true;
      if (owner) line_contract(0, acc, dummy);
      if (role == 1 || role == 2) publish(acc);
      __syncthreads();
      if (role == 0) {
        // rate of the x-line at every i -> pushed to the CTA owning x-plane i
#pragma unroll
        for (int i = 0; i < P; ++i)
#pragma unroll
          for (int v = 0; v < M; ++v) {
            const double r = (-acc[i][v] - B1[xrow + i * M + v]) - B2[xrow + i * M + v];
            push(G + xrow + c * M + v, i, barG, r);
          }
      }
      // time operator for the nodes of x-plane c at every time
      // node (c, a0, b0): the three owners of (a0, b0) split its P times
      double sd = 0.0, sq = 0.0;
      if (owner) {
        wait(barG, phG);
        double r[P][M];
#pragma unroll
        for (int s = 0; s < P; ++s)
#pragma unroll
          for (int v = 0; v < M; ++v) r[s][v] = G[xrow + s * M + v];
#pragma unroll
        for (int t = 0; t < P; ++t) {
          if (t < tlo || t >= thi) continue;
          double* qo = B3 + xrow + t * M;   // previous iterate of (node, t), local
          const double g0 = T.g0[t];
#pragma unroll
          for (int v = 0; v < M; ++v) {
            double cc = 0.0;
#pragma unroll
            for (int s = 0; s < P; ++s) cc = fma(T.gw[t * P + s], r[s][v], cc);
            const double qn = cc * dt + g0 * uu[v];
            const double dq = qo[v] - qn;
            sd = fma(dq, dq, sd);
            sq = fma(qn, qn, sq);
            qo[v] = qn;
            push(Q + qnode + v, t, barQ, qn);
          }
        }
      }
      phG ^= 1;
      // residual: warp trees, warps in order, CTAs in order (every CTA gets
      // the same partials and folds them in the same order -> one decision)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sd += __shfl_xor_sync(0xffffffffu, sd, o);
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
      }
      if (lane == 0) {
        red[2 * warp] = sd;
        red[2 * warp + 1] = sq;
      }
      __syncthreads();
      if (tid < C::C) {
        double t1 = 0.0, t2 = 0.0;
        for (int w = 0; w < NW; ++w) {
          t1 += red[2 * w];
          t2 += red[2 * w + 1];
        }
        push(credg + 2 * c, tid, barC, t1);
        push(credg + 2 * c + 1, tid, barC, t2);
      }
      wait(barQ, phQ);
      wait(barC, phC);
      phQ ^= 1;
      phC ^= 1;
      double t1 = 0.0, t2 = 0.0;
#pragma unroll
      for (int s = 0; s < C::C; ++s) {
        t1 += credg[2 * s];
        t2 += credg[2 * s + 1];
      }
      const double res = T.k1_opnorm * sqrt(t1);
      const double scale = 1.0 + sqrt(t2);
      conv = res <= a.tol * scale;
      nsw = it + 1;
      if (conv && it + 1 >= a.min_iter) fz = true;
    }

    // ---------------- traces, admissibility, volume ---------------------
    bool ok = true;
    {
      double acc[P][M];
      if (owner) {
        // face traces of the line at time c (face-kernel block layouts:
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
        const int pos = role == 0 ? (a0 * P + b0) * P + c
                                  : (role == 1 ? (b0 * P + c) * P + a0 : (c * P + a0) * P + b0);
        const size_t fs = (size_t)a.n_elem * C::TB;
        double* tlo = a.traces + (size_t)(2 * dir) * fs + (size_t)e * C::TB + (size_t)pos * M;
        double* thi = tlo + fs;
#pragma unroll
        for (int v = 0; v < M; ++v) {
          tlo[v] = lo[v];
          thi[v] = hi[v];
        }
        line_contract(1, acc, ok);
      }
      if (role == 1 || role == 2) publish(acc);
      if (a.q_out) {
        for (int x = tid; x < PD; x += NT) {
          const int i = x / PP, j = (x / P) % P, k = x % P;
#pragma unroll
          for (int v = 0; v < M; ++v)
            a.q_out[(((size_t)e * PD + x) * P + c) * M + v] = Q[i * SI + j * SJ + k * M + v];
        }
      }
      if (tid == 0) {
        mbar_expect_tx(barG, PD * M * 8);   // volume parts of x-plane c from every slice
        mbar_expect_tx(barF, C::C * 8);     // verdicts
      }
      const int all_ok = __syncthreads_and(ok ? 1 : 0);
      // Q is dead for this element: fetch the next element's u^n
      if (e + ncl < a.n_elem) fetch_u(e + ncl);
      if (role == 0) {
        // this slice's volume part at the x-line's nodes (i, a0, b0):
        // w_c sum_dir scale_dir(node) stiff x_dir F_dir(q_c)
        const double wa = T.weights[a0], wb = T.weights[b0];
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const double wi = T.weights[i];
          const double s0 = sc0 * (wa * wb), s1 = sc1 * (wi * wb), s2 = sc2 * (wi * wa);
#pragma unroll
          for (int v = 0; v < M; ++v) {
            double vv = s0 * acc[i][v];
            vv += s1 * B1[xrow + i * M + v];
            vv += s2 * B2[xrow + i * M + v];
            push(G + xrow + c * M + v, i, barG, wtc * vv);
          }
        }
      }
      if (tid < C::C) push(okg + c, tid, barF, all_ok ? 1.0 : 0.0);
    }
    if (node_role) {
      // vol(node) = sum over slices in slice order
      wait(barG, phG);
      double* out = a.vol + ((size_t)e * PD + nnode) * M;
#pragma unroll
      for (int v = 0; v < M; ++v) {
        double vsum = 0.0;
#pragma unroll
        for (int s = 0; s < C::C; ++s) vsum += G[xrow + s * M + v];
        out[v] = vsum;
      }
    }
    phG ^= 1;
    if (tid == 0) {
      wait(barF, phF);
      if (c == 0) {
        int okall = 1;
        for (int s = 0; s < C::C; ++s) okall &= okg[s] != 0.0;
        a.pred_bad[e] = (conv ? 0 : ADG_PRED_NOT_CONVERGED) | (okall ? 0 : ADG_PRED_INADMISSIBLE);
        a.sweeps[e] = nsw ? nsw : it;
      }
    }
    phF ^= 1;
  }
  cluster_barrier();   // no CTA leaves while a push to its shared memory may be in flight
}

template <int P>
static int launch_cluster(const ClArgs& a, cudaStream_t st, int num_sms, std::string* err) {
  using C = ClCfg<P>;
  auto kern = predict_cluster_kernel<P>;
  static PerDevice attr;
  if (attr.first()) {
    cudaError_t ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)C::SMEM);
    if (ce == cudaSuccess && C::C > 8)
      ce = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (ce != cudaSuccess) {
      *err = cudaGetErrorString(ce);
      return ADG_ERR_CUDA;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C::C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(C::NT);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C::C * 1024);
  int max_cl = 0;
  cudaError_t ce = cudaOccupancyMaxActiveClusters(&max_cl, kern, &cfg);
  if (ce != cudaSuccess || max_cl < 1) {
    *err = ce != cudaSuccess ? cudaGetErrorString(ce) : "cluster predictor cannot be scheduled";
    return ADG_ERR_CUDA;
  }
  const int64_t ncl = std::min<int64_t>(a.n_elem, (int64_t)max_cl);
  if (ncl < 1) return ADG_OK;
  cfg.gridDim = dim3((unsigned)(ncl * C::C));
  ce = cudaLaunchKernelEx(&cfg, kern, a);
  if (ce == cudaSuccess) ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    *err = cudaGetErrorString(ce);
    return ADG_ERR_CUDA;
  }
  (void)num_sms;
  return ADG_OK;
}

bool predict_cluster_supported(const adg_grid* g) {
  return g->dim == 3 && g->degree >= 7 && g->degree <= 9 && g->mode != ADG_MODE_PRIMITIVE;
}

int predict_cluster(const adg_grid* g, const double* u, const double* dt_dev, double tol,
                    int max_iter, int min_iter, double* q_out, double* vol, double* traces,
                    uint8_t* pred_bad, int32_t* sweeps, cudaStream_t st, int num_sms,
                    std::string* err) {
  ClArgs a{};
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
    case 8: return launch_cluster<8>(a, st, num_sms, err);
    case 9: return launch_cluster<9>(a, st, num_sms, err);
    case 10: return launch_cluster<10>(a, st, num_sms, err);
  }
  *err = "cluster predictor: unsupported degree";
  return ADG_ERR_UNSUPPORTED;
}

}  // namespace adg
