// Viscous condensed-operator kernels in point form (K7, second generation).
//
// Viscous couplings of the condensed operator and the S correction
// (reference assembly.py:772-976 and :1037-1173), organised so that every
// chain "trace / local unknowns -> Y (NN x 15) -> M^-1 -> value at a point"
// is a single contraction with a precomputed point table (ViscGeo::cxt,
// dzt, pmt, tpp; built once at context creation):
//   yq(pt)[t][b] = (1/det) [ sum_k area_k n_k,b sum_jj CX_k[pt][jj] x_k[jj][t]
//                          + sum_j PM[pt][j] r_q[j][t][b] ]
//                 + sum_k2 Jinv[k2][b] sum_i DZ_k2[pt][i] z[i][t]
// with PM = phi_pt Mref^-1, CX_k = -PM R_k Eref_k, DZ_k2 = PM Kref_k2.
// One thread owns one quadrature point (volume points first, then the four
// faces' points), so the G(w, yq) evaluations of a macro run in one pass
// instead of a sequence of shared-memory phases; register blocking cuts the
// shared-memory traffic per FMA that bounded the first generation.
#pragma once
#include "mhdg_viscous.cuh"

namespace mhdg {

// Row stride of the nodal 5-vectors (w, x, z) in shared memory: 16-byte rows,
// read as two LDS.128 + one LDS.64 instead of five LDS.64.  The point loops
// issue one such row per FMA group of five and were bound by the shared-
// memory instruction rate (six loads per five FMAs), not by the FP64 pipe.
constexpr int VRS = 6;
MHDG_DEV void vf_ld5(const double* __restrict__ row, double (&v)[5]) {
  const double2 a = *reinterpret_cast<const double2*>(row);
  const double2 b = *reinterpret_cast<const double2*>(row + 2);
  v[0] = a.x;
  v[1] = a.y;
  v[2] = b.x;
  v[3] = b.y;
  v[4] = row[4];
}

template <int P>
struct VFast {
  using D = Dims<P>;
  static constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF, NM = D::NM;
  static constexpr int NPT = NQ + 4 * NQF;
  static constexpr int NT = 128;
  // in-kernel: macros per CTA (one thread per point)
  static constexpr int MBI = NPT <= 32 ? 4 : (NPT <= 64 ? 2 : 1);
  static constexpr int SPI = NT / MBI;                 // thread slots per macro
  // out-kernel: face points only
  static constexpr int NPF = 4 * NQF;
  static constexpr int MBO = NT / NPF;
  static constexpr int NK = 3 * NQ + 4 * NQF;          // test entries (vol (q,kk) + face pts)
  static constexpr int NKP = (NK + 3) / 4 * 4;          // padded to the DMMA k-step
  static constexpr int NTI = (NN + 7) / 8;              // 8-wide node tiles
  static constexpr int WPM = SPI / 32;                  // warps per macro (in-kernel)
  // CTA = NG independent groups of GT threads (named barriers), one per
  // former CTA: the groups drift in phase against each other like separate
  // CTAs, while the point tables are staged ONCE per CTA in shared memory.
  // Read through L1 they missed a quarter of the time (111 KB of tables at
  // k = 3 against the streaming w / x / tensor traffic: ncu L1 hit rate 74%,
  // long-scoreboard stalls 4.1 per issue, issue slots 27% busy).
  static constexpr int GT = NT, NG = 4, CT = NG * GT;
  // test-table row stride in shared memory: >= NN and = 4 (mod 16), so the
  // B-fragment reads (lane = 4 n + kk -> word kk * TS + n) hit 32 distinct
  // banks (the global table's stride NTI * 8 = 24 gave two-way conflicts)
  static constexpr int TS = NN + ((4 - NN) % 16 + 16) % 16;
  static constexpr int T_PHIT = NN * NPT, T_CXT = 4 * NFN * NPT, T_TST = NKP * TS;
  static constexpr int IN_TAB = T_PHIT + T_CXT + T_TST + NQF * NFN;   // + fphi
  static constexpr int MT = (NPF + 7) / 8, KX = (NFN + 3) / 4, KZ = (NN + 3) / 4;
  static constexpr int TM = (NFN + 7) / 8, TK = (NQF + 3) / 4;
  static constexpr int T_CXF = 4 * MT * KX * 32, T_DZF = 3 * MT * KZ * 32, T_FPF = TM * TK * 32,
                       T_PF = 4 * NQF * NFN, T_FPHI = NQF * NFN;
  static constexpr int OUT_TAB = T_CXF + T_DZF + T_FPF + T_PF + T_FPHI;
  static constexpr int META = 8 + 4 * NFN;   // Geo::meta row: face ids (4), trace permutations (4 NFN), flags (4)
  // w / x / geometry of a macro arrive by cp.async one macro ahead (two
  // buffers); the face ids / permutations the x gather needs, two ahead
  struct In {
    alignas(16) double W[2][NN * VRS], X[2][4 * NFN * VRS];
    double RQ[NN * 15], Gk[NKP * 5], part[WPM][NTI * 8 * 8], geo[2][26];
    int meta[2][META];
  };
  // out-kernel: the same pipeline; the face ids live in a ring of three (the
  // trace scatter at the end of macro i still reads meta(i) while meta(i + 2)
  // arrives); r_q (condensed rhs only) shares YQ (matvec only)
  struct Out {
    alignas(16) double W[2][NN * VRS], Z[2][NN * VRS], X[2][4 * NFN * VRS];
    double Gf[NPF * 5], YQ[NPF * 15 > NN * 15 ? NPF * 15 : NN * 15], geo[2][26];
    int meta[3][META];
  };
  static_assert(IN_TAB % 2 == 0 && OUT_TAB % 2 == 0, "16-byte alignment of the per-group structs");
  static constexpr size_t in_bytes = (size_t)IN_TAB * 8 + sizeof(In) * MBI * NG;
  static constexpr size_t out_bytes = (size_t)OUT_TAB * 8 + sizeof(Out) * MBO * NG + 4 * NFN * sizeof(int);
};

// yq contribution of the trace: (area_k n_k,b) sum_jj CX_k[pt][jj] x_k[jj][t]
template <int P>
MHDG_DEV void vf_add_x(const double* __restrict__ cxt, int pt, const double* X, const double* geo, double yq[5][3]) {
  constexpr int NFN = Dims<P>::NFN, NPT = VFast<P>::NPT;
#pragma unroll 1
  for (int k = 0; k < 4; ++k) {
    double u[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int jj = 0; jj < NFN; ++jj) {
      const double c = cxt[(k * NFN + jj) * NPT + pt];
      double xr[5];
      vf_ld5(X + (k * NFN + jj) * VRS, xr);
#pragma unroll
      for (int t = 0; t < 5; ++t) u[t] += c * xr[t];
    }
    const double a = geo[22 + k];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double an = a * geo[10 + k * 3 + b];
#pragma unroll
      for (int t = 0; t < 5; ++t) yq[t][b] += an * u[t];
    }
  }
}

template <int P>
MHDG_DEV void vf_add_rq(const ViscGeo& vg, int pt, const double* RQ, double yq[5][3]) {
  constexpr int NN = Dims<P>::NN, NPT = VFast<P>::NPT;
#pragma unroll 4
  for (int j = 0; j < NN; ++j) {
    const double c = __ldg(vg.pmt + (size_t)j * NPT + pt);
#pragma unroll
    for (int t = 0; t < 5; ++t)
#pragma unroll
      for (int b = 0; b < 3; ++b) yq[t][b] += c * RQ[j * 15 + t * 3 + b];
  }
}

template <int P>
MHDG_DEV void vf_add_z(const ViscGeo& vg, int pt, const double* Z, const double* geo, double yq[5][3]) {
  constexpr int NN = Dims<P>::NN, NPT = VFast<P>::NPT;
#pragma unroll 1
  for (int k2 = 0; k2 < 3; ++k2) {
    double u[5] = {0, 0, 0, 0, 0};
#pragma unroll 4
    for (int i = 0; i < NN; ++i) {
      const double c = __ldg(vg.dzt + (size_t)(k2 * NN + i) * NPT + pt);
#pragma unroll
      for (int t = 0; t < 5; ++t) u[t] += c * Z[i * VRS + t];
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double jb = geo[1 + k2 * 3 + b];
#pragma unroll
      for (int t = 0; t < 5; ++t) yq[t][b] += jb * u[t];
    }
  }
}

// ---------------------------------------------------------------------------
// k_visc_in2: g = -r_w[1,2] - vvhat(x)[0,2] + vq(M^-1 (r_q[1,2] + qvhat(x)[0,2]))
//   (mode 0 matvec, 1 condensed rhs, 2 recovery)
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(VFast<P>::CT, 1)
k_visc_in2(Geo g, ViscGeo vg, int mode, const double* __restrict__ wlin, const double* __restrict__ hhat,
           const double* __restrict__ x, const double* __restrict__ r_w, const double* __restrict__ r_q,
           double* __restrict__ gout) {
  using V = VFast<P>;
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF, NM = D::NM, NPT = V::NPT;
  constexpr int MB = V::MBI, SP = V::SPI, NK = V::NK;
  extern __shared__ __align__(16) double smem[];
  double* sPHIT = smem;                  // (NN, NPT)
  double* sCXT = sPHIT + V::T_PHIT;      // (4 NFN, NPT)
  double* sTST = sCXT + V::T_CXT;        // (NKP, TS)
  double* sFPHI = sTST + V::T_TST;       // (NQF, NFN)
  const int grp = threadIdx.x / V::GT, tid = threadIdx.x % V::GT, slot = tid / SP, lt = tid % SP;
  typename V::In* sm = reinterpret_cast<typename V::In*>(sFPHI + NQF * NFN) + grp * MB;
  const double gam = g.gamma;
  const bool use_x = mode != 1, use_r = mode != 0;
  const int nblk = (g.E + MB - 1) / MB;
  for (int i = threadIdx.x; i < V::T_PHIT; i += V::CT) sPHIT[i] = vg.phit[i];
  for (int i = threadIdx.x; i < V::T_CXT; i += V::CT) sCXT[i] = vg.cxt[i];
  for (int i = threadIdx.x; i < V::NKP * NN; i += V::CT) sTST[(i / NN) * V::TS + i % NN] = vg.tst[(i / NN) * (V::NTI * 8) + i % NN];
  for (int i = threadIdx.x; i < NQF * NFN; i += V::CT) sFPHI[i] = g.fphi[i];
  for (int i = NK * 5 + lt; i < V::NKP * 5; i += SP) sm[slot].Gk[i] = 0.0;
  __syncthreads();
  auto gsync = [&]() { group_sync(1 + grp, V::GT); };
  pdl_wait();   // before: immutable point tables into shared memory, padding (mhdg_kernels.cuh PDL invariant)
  // Software pipeline per group (the load phase and the barrier behind it
  // were 38% of the stall samples: two dependent global round trips per
  // macro with nothing to overlap them but the other three groups):
  //   top of macro i:  data(i) and meta(i + 1) have landed
  //                    issue data(i + 1) (its x gather reads meta(i + 1)),
  //                    issue meta(i + 2), prefetch hhat(i + 1) towards L2
  //   then compute macro i from buffer i & 1.
  typename V::In& S = sm[slot];
  const int bstride = gridDim.x * V::NG;
  auto issue_meta = [&](int blkn, int buf) {
    const int en = blkn * MB + slot;
    if (blkn < nblk && en < g.E)
      for (int i = lt; i < V::META; i += SP) cp_async4(&S.meta[buf][i], g.meta + (size_t)en * V::META + i);
  };
  auto issue_data = [&](int blkn, int buf) {
    const int en = blkn * MB + slot;
    if (blkn >= nblk || en >= g.E) return;
    for (int i = lt; i < NN * 5; i += SP)
      cp_async8(&S.W[buf][(i / 5) * VRS + i % 5], wlin + (size_t)en * NN * 5 + i);
    for (int i = lt; i < 26; i += SP) cp_async8(&S.geo[buf][i], g.geo26 + (size_t)en * 50 + i);
    if (use_x) {
      const int* mt = S.meta[buf];
      for (int i = lt; i < 4 * NFN * 5; i += SP) {
        const int k = i / (NFN * 5), j = (i / 5) % NFN, s2 = i % 5;
        cp_async8(&S.X[buf][(i / 5) * VRS + s2], x + ((size_t)mt[k] * NFN + mt[4 + k * NFN + j]) * 5 + s2);
      }
      // 25 x NQF doubles per face, contiguous per (macro, face)
      for (int i = lt * 16; i < 4 * 25 * NQF; i += SP * 16) prefetch_l2(hhat + (size_t)en * 4 * 25 * NQF + i);
    }
  };
  int blk = blockIdx.x * V::NG + grp;
  issue_meta(blk, 0);
  cp_async_wait_all();
  gsync();
  issue_data(blk, 0);
  issue_meta(blk + bstride, 1);
  for (int cur = 0; blk < nblk; blk += bstride, cur ^= 1) {
    const int e = blk * MB + slot;
    const bool live = e < g.E;
    cp_async_wait_all();
    gsync();
    issue_data(blk + bstride, cur ^ 1);
    issue_meta(blk + 2 * bstride, cur);
    if (use_r) {
      if (live)
        for (int i = lt; i < NN * 15; i += SP) S.RQ[i] = r_q[(size_t)e * NN * 15 + i];
      gsync();
    }
    const double* sW = S.W[cur];
    const double* sX = S.X[cur];
    const double* sGeo = S.geo[cur];
    if (live && lt < NPT) {
      const int pt = lt;
      double wq[5] = {0, 0, 0, 0, 0}, yq[5][3];
#pragma unroll
      for (int t = 0; t < 5; ++t) yq[t][0] = yq[t][1] = yq[t][2] = 0.0;
#pragma unroll 4
      for (int i = 0; i < NN; ++i) {
        const double a = sPHIT[i * NPT + pt];
        double wr[5];
        vf_ld5(sW + i * VRS, wr);
#pragma unroll
        for (int t = 0; t < 5; ++t) wq[t] += a * wr[t];
      }
      if (use_x) vf_add_x<P>(sCXT, pt, sX, sGeo, yq);
      if (use_r) vf_add_rq<P>(vg, pt, S.RQ, yq);
      const double idet = 1.0 / sGeo[0];
#pragma unroll
      for (int t = 0; t < 5; ++t)
#pragma unroll
        for (int b = 0; b < 3; ++b) yq[t][b] *= idet;
      double u[5], Gv[5][3];
      to_conservative(wq, g.form, gam, u);
      visc_G(vg, g.form, wq, u, yq, gam, Gv);
      if (pt < NQ) {
        const double vw = g.qw[pt] * sGeo[0];
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const double j0 = sGeo[1 + kk * 3], j1 = sGeo[2 + kk * 3], j2 = sGeo[3 + kk * 3];
#pragma unroll
          for (int t = 0; t < 5; ++t)
            S.Gk[(pt * 3 + kk) * 5 + t] = -(vw * ((j0 * Gv[t][0] + j1 * Gv[t][1]) + j2 * Gv[t][2]));
        }
      } else {
        const int it = pt - NQ, k = it / NQF, qp = it % NQF;
        const double fwq = g.fw[qp] * sGeo[22 + k];
        const double n0 = sGeo[10 + k * 3], n1 = sGeo[11 + k * 3], n2 = sGeo[12 + k * 3];
        double hx[5] = {0, 0, 0, 0, 0};
        if (use_x) {
          double xq[5] = {0, 0, 0, 0, 0};
#pragma unroll
          for (int j = 0; j < NFN; ++j) {
            const double b2 = sFPHI[qp * NFN + j];
            double xr[5];
            vf_ld5(sX + (k * NFN + j) * VRS, xr);
#pragma unroll
            for (int t = 0; t < 5; ++t) xq[t] += b2 * xr[t];
          }
          const double* h = hhat + ((size_t)e * 4 + k) * 25 * NQF + qp;   // (E,4,25,NQF)
#pragma unroll
          for (int s2 = 0; s2 < 5; ++s2) {
            double a = 0.0;
#pragma unroll
            for (int t = 0; t < 5; ++t) a += h[(s2 * 5 + t) * NQF] * xq[t];
            hx[s2] = a;
          }
        }
#pragma unroll
        for (int t = 0; t < 5; ++t)
          S.Gk[(3 * NQ + it) * 5 + t] = fwq * (((Gv[t][0] * n0 + Gv[t][1] * n1) + Gv[t][2] * n2) - hx[t]);
      }
    }
    gsync();
    // tests on the FP64 tensor cores: gout^T (5 x NN) = Gk^T (5 x NK) . TST (NK x NN),
    // K split across the macro's warps, partials summed in warp order
    {
      constexpr int KS = V::NKP / 4, NTI = V::NTI, WPM = V::WPM;
      const int wl = lt >> 5, lane = tid & 31;
      const int ks0 = wl * KS / WPM, ks1 = (wl + 1) * KS / WPM;
      double c[NTI][2];
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) c[nt][0] = c[nt][1] = 0.0;
      const int sa = lane >> 2, kl = lane & 3;
      for (int ks = ks0; ks < ks1; ++ks) {
        const int K = ks * 4 + kl;
        const double a = sa < 5 ? S.Gk[K * 5 + sa] : 0.0;
#pragma unroll
        for (int nt = 0; nt < NTI; ++nt)
          dmma_8x8x4(c[nt], a, nt * 8 + (lane >> 2) < NN ? sTST[K * V::TS + nt * 8 + (lane >> 2)] : 0.0);
      }
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        S.part[wl][(nt * 8 + kl * 2) * 8 + sa] = c[nt][0];
        S.part[wl][(nt * 8 + kl * 2 + 1) * 8 + sa] = c[nt][1];
      }
    }
    gsync();
    if (live)
      for (int o = lt; o < NM; o += SP) {
        const int i = o / 5, s2 = o % 5;
        double acc = S.part[0][i * 8 + s2];
#pragma unroll
        for (int w2 = 1; w2 < V::WPM; ++w2) acc += S.part[w2][i * 8 + s2];
        gout[(size_t)e * NM + o] = use_r ? (-r_w[(size_t)e * NM + o] + acc) : acc;
      }
  }
}

// ---------------------------------------------------------------------------
// k_visc_out2: y += hh x[0] + hw z - vhatq(M^-1 (qv z + qvhat(x)[0] + r_q[1]))
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(VFast<P>::CT, 1)
k_visc_out2(Geo g, ViscGeo vg, int mode, const double* __restrict__ wlin, const double* __restrict__ hh,
            const double* __restrict__ hw, const double* __restrict__ x, const double* __restrict__ z,
            const double* __restrict__ r_q, double* __restrict__ y) {
  using V = VFast<P>;
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF, NM = D::NM;
  constexpr int MB = V::MBO, NPF = V::NPF;
  extern __shared__ __align__(16) double smem[];
  double* sCXF = smem;                   // fragment-ordered CX slices
  double* sDZF = sCXF + V::T_CXF;        // fragment-ordered DZ slices
  double* sFPF = sDZF + V::T_DZF;        // fragment-ordered fphi
  double* sPF = sFPF + V::T_FPF;         // (4 NQF, NFN)
  double* sFPHI = sPF + V::T_PF;         // (NQF, NFN)
  const int grp = threadIdx.x / V::GT, tid = threadIdx.x % V::GT;
  typename V::Out* sm = reinterpret_cast<typename V::Out*>(sFPHI + V::T_FPHI) + grp * MB;
  int* sRows = reinterpret_cast<int*>(reinterpret_cast<typename V::Out*>(sFPHI + V::T_FPHI) + V::NG * MB);
  const int slot = tid / NPF, lt = tid % NPF;
  const double gam = g.gamma;
  const int nblk = (g.E + MB - 1) / MB;
  for (int i = threadIdx.x; i < V::T_CXF; i += V::CT) sCXF[i] = vg.cxf[i];
  for (int i = threadIdx.x; i < V::T_DZF; i += V::CT) sDZF[i] = vg.dzf[i];
  for (int i = threadIdx.x; i < V::T_FPF; i += V::CT) sFPF[i] = vg.fpf[i];
  for (int i = threadIdx.x; i < V::T_PF; i += V::CT) sPF[i] = g.pf[i];
  for (int i = threadIdx.x; i < V::T_FPHI; i += V::CT) sFPHI[i] = g.fphi[i];
  for (int i = threadIdx.x; i < 4 * NFN; i += V::CT) sRows[i] = g.rows[i];
  __syncthreads();
  auto gsync = [&]() { group_sync(1 + grp, V::GT); };
  pdl_wait();   // before: immutable point tables into shared memory (mhdg_kernels.cuh PDL invariant)
  // software pipeline as in k_visc_in2: data(i + 1) and meta(i + 2) are in
  // flight while macro i is computed; hw / hh of macro i + 1 go towards L2
  typename V::Out& S = sm[slot < MB ? slot : 0];
  const int bstride = gridDim.x * V::NG;
  auto issue_meta = [&](int blkn, int ms) {
    const int en = blkn * MB + slot;
    if (slot < MB && blkn < nblk && en < g.E)
      for (int i = lt; i < V::META; i += NPF) cp_async4(&S.meta[ms][i], g.meta + (size_t)en * V::META + i);
  };
  auto issue_data = [&](int blkn, int buf, int ms) {
    const int en = blkn * MB + slot;
    if (slot >= MB || blkn >= nblk || en >= g.E) return;
    for (int i = lt; i < NN * 5; i += NPF) {
      cp_async8(&S.W[buf][(i / 5) * VRS + i % 5], wlin + (size_t)en * NN * 5 + i);
      cp_async8(&S.Z[buf][(i / 5) * VRS + i % 5], z + (size_t)en * NM + i);
    }
    for (int i = lt; i < 26; i += NPF) cp_async8(&S.geo[buf][i], g.geo26 + (size_t)en * 50 + i);
    if (mode == 0) {
      const int* mt = S.meta[ms];
      for (int i = lt; i < 4 * NFN * 5; i += NPF) {
        const int k = i / (NFN * 5), j = (i / 5) % NFN, s2 = i % 5;
        cp_async8(&S.X[buf][(i / 5) * VRS + s2], x + ((size_t)mt[k] * NFN + mt[4 + k * NFN + j]) * 5 + s2);
      }
    }
    for (int i = lt * 16; i < 4 * 25 * NQF; i += NPF * 16) {
      prefetch_l2(hw + (size_t)en * 4 * 25 * NQF + i);
      if (mode == 0) prefetch_l2(hh + (size_t)en * 4 * 25 * NQF + i);
    }
  };
  int blk = blockIdx.x * V::NG + grp;
  issue_meta(blk, 0);
  cp_async_wait_all();
  gsync();
  issue_data(blk, 0, 0);
  issue_meta(blk + bstride, 1);
  for (int cur = 0, mc = 0; blk < nblk; blk += bstride, cur ^= 1, mc = (mc + 1) % 3) {
    const int e = blk * MB + slot;
    const bool live = slot < MB && e < g.E;
    cp_async_wait_all();
    gsync();
    issue_data(blk + bstride, cur ^ 1, (mc + 1) % 3);
    issue_meta(blk + 2 * bstride, (mc + 2) % 3);
    if (mode == 1) {
      if (live)
        for (int i = lt; i < NN * 15; i += NPF) S.YQ[i] = r_q[(size_t)e * NN * 15 + i];
      gsync();
    }
    if (mode == 0) {
      // gradient unknowns at the face points on the FP64 tensor cores, per
      // (macro slot, 8-point tile):
      //   yq = (1/det) sum_k (area n)_k (CX_k x_k) + sum_k2 Jinv[k2] (DZ_k2 z)
      // (the point-per-thread contraction spent one shared-memory load per
      // FMA on the broadcast x / z values)
      constexpr int MT = V::MT, KX = V::KX, KZ = V::KZ;
      const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, nn = lane >> 2;
      for (int job = warp; job < MB * MT; job += V::GT / 32) {
        const int sl = job / MT, mt = job % MT;
        if (blk * MB + sl >= g.E) continue;
        typename V::Out& Sx = sm[sl];
        double acc[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double c[2] = {0.0, 0.0};
#pragma unroll
          for (int ks = 0; ks < KX; ++ks) {
            const int jj = ks * 4 + kq;
            const double b = (jj < NFN && nn < 5) ? Sx.X[cur][(k * NFN + jj) * VRS + nn] : 0.0;
            dmma_8x8x4(c, sCXF[((k * MT + mt) * KX + ks) * 32 + lane], b);
          }
          const double a = Sx.geo[cur][22 + k];
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const double an = a * Sx.geo[cur][10 + k * 3 + b];
            acc[0][b] += an * c[0];
            acc[1][b] += an * c[1];
          }
        }
        const double idet = 1.0 / Sx.geo[cur][0];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
          for (int b = 0; b < 3; ++b) acc[h2][b] *= idet;
#pragma unroll
        for (int k2 = 0; k2 < 3; ++k2) {
          double c[2] = {0.0, 0.0};
#pragma unroll
          for (int ks = 0; ks < KZ; ++ks) {
            const int i = ks * 4 + kq;
            const double b = (i < NN && nn < 5) ? Sx.Z[cur][i * VRS + nn] : 0.0;
            dmma_8x8x4(c, sDZF[((k2 * MT + mt) * KZ + ks) * 32 + lane], b);
          }
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const double jb = Sx.geo[cur][1 + k2 * 3 + b];
            acc[0][b] += jb * c[0];
            acc[1][b] += jb * c[1];
          }
        }
        const int pt2 = mt * 8 + nn;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int t = kq * 2 + h2;
          if (t < 5 && pt2 < NPF)
#pragma unroll
            for (int b = 0; b < 3; ++b) Sx.YQ[pt2 * 15 + t * 3 + b] = acc[h2][b];
        }
      }
      gsync();
    }
    if (live) {
      const int it = lt, k = it / NQF, qp = it % NQF, pt = NQ + it;
      double wq[5] = {0, 0, 0, 0, 0}, zq[5] = {0, 0, 0, 0, 0}, xq[5] = {0, 0, 0, 0, 0}, yq[5][3];
#pragma unroll
      for (int t = 0; t < 5; ++t) yq[t][0] = yq[t][1] = yq[t][2] = 0.0;
#pragma unroll
      for (int j = 0; j < NFN; ++j) {
        const double a = sPF[it * NFN + j];
        const int row = sRows[k * NFN + j];
        double wr[5], zr[5];
        vf_ld5(S.W[cur] + row * VRS, wr);
        vf_ld5(S.Z[cur] + row * VRS, zr);
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          wq[t] += a * wr[t];
          zq[t] += a * zr[t];
        }
        if (mode == 0) {
          const double b2 = sFPHI[qp * NFN + j];
          double xr[5];
          vf_ld5(S.X[cur] + (k * NFN + j) * VRS, xr);
#pragma unroll
          for (int t = 0; t < 5; ++t) xq[t] += b2 * xr[t];
        }
      }
      if (mode == 0) {
#pragma unroll
        for (int t = 0; t < 5; ++t)
#pragma unroll
          for (int b = 0; b < 3; ++b) yq[t][b] = S.YQ[it * 15 + t * 3 + b];
      } else {
        if (mode == 1) vf_add_rq<P>(vg, pt, S.YQ, yq);
        const double idet = 1.0 / S.geo[cur][0];
#pragma unroll
        for (int t = 0; t < 5; ++t)
#pragma unroll
          for (int b = 0; b < 3; ++b) yq[t][b] *= idet;
        vf_add_z<P>(vg, pt, S.Z[cur], S.geo[cur], yq);
      }
      double u[5], Gv[5][3];
      to_conservative(wq, g.form, gam, u);
      visc_G(vg, g.form, wq, u, yq, gam, Gv);
      const double fwq = g.fw[qp] * S.geo[cur][22 + k];
      const double n0 = S.geo[cur][10 + k * 3], n1 = S.geo[cur][11 + k * 3], n2 = S.geo[cur][12 + k * 3];
      const size_t base = ((size_t)e * 4 + k) * 25 * NQF + qp;   // (E,4,25,NQF)
#pragma unroll
      for (int s2 = 0; s2 < 5; ++s2) {
        double a = 0.0, b2 = 0.0;
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          a += hw[base + (s2 * 5 + t) * NQF] * zq[t];
          if (mode == 0) b2 += hh[base + (s2 * 5 + t) * NQF] * xq[t];
        }
        const double gn = (Gv[s2][0] * n0 + Gv[s2][1] * n1) + Gv[s2][2] * n2;
        S.Gf[it * 5 + s2] = fwq * b2 + (fwq * a - fwq * gn);
      }
    }
    gsync();
    // trace tests on DMMA, per (macro slot, face): C[j][s] = sum_qp fphi[qp][j] Gf[qp][s]
    // (A fragments of fphi from the fragment-ordered table fpf, staged in shared memory)
    {
      constexpr int TM = V::TM, TK = V::TK;
      const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, nn = lane >> 2;
      for (int job = warp; job < MB * 4; job += V::GT / 32) {
        const int sl = job / 4, k = job % 4;
        if (blk * MB + sl >= g.E) continue;
        const typename V::Out& Sx = sm[sl];
        double c[TM][2];
#pragma unroll
        for (int t = 0; t < TM; ++t) c[t][0] = c[t][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < TK; ++ks) {
          const int qp = ks * 4 + kq;
          const double b = (qp < NQF && nn < 5) ? Sx.Gf[(k * NQF + qp) * 5 + nn] : 0.0;
#pragma unroll
          for (int t = 0; t < TM; ++t) dmma_8x8x4(c[t], sFPF[(t * TK + ks) * 32 + lane], b);
        }
#pragma unroll
        for (int t = 0; t < TM; ++t)
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int j = t * 8 + nn, s2 = kq * 2 + h2;
            if (j < NFN && s2 < 5)
              atomicAdd(&y[((size_t)Sx.meta[mc][k] * NFN + Sx.meta[mc][4 + k * NFN + j]) * 5 + s2], c[t][h2]);
          }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_visc_scorr2: S[(i,s),(j,t)] -= sum_K TST[K][i] sum_b C[K][s][t,b] Phi_b[pt(K)][j]
//   K = (q, kk) volume entries (TST = dphi_kk, C = -vw Jinv[kk] . dG/dq)
//     + face points (TST = phi_face at face rows, C = fw dG/dq . n),
//   Phi_b[pt][j] = sum_k2 Jinv[k2][b] (phi_pt Pref_k2)[pt][j]  (= phi_pt M_e^-1 K_e,b).
// Thread = (s, t, pair of j) with all NN rows i in registers.
// ---------------------------------------------------------------------------
template <int P>
struct SCorr2 {
  using D = Dims<P>;
  static constexpr int NN = D::NN, NQ = D::NQ, NQF = D::NQF;
  static constexpr int NPT = NQ + 4 * NQF;
  static constexpr int NT = 256;
  static constexpr int JG = 2;
  static constexpr int NJG = (NN + JG - 1) / JG;
  static constexpr int CH = 32;                       // points per chunk
  static constexpr size_t bytes = (size_t)(CH * 3 * 75 + CH * 10 + NN * 5 + 16) * 8;
};

template <int P>
__global__ void __launch_bounds__(256, (P >= 3 ? 1 : 2))
k_visc_scorr2(Geo g, ViscGeo vg, const double* __restrict__ w, double* __restrict__ S) {
  using D = Dims<P>;
  using SC = SCorr2<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NQF = D::NQF, NM = D::NM, NPT = SC::NPT, CH = SC::CH;
  constexpr int JG = SC::JG, NJG = SC::NJG;
  extern __shared__ __align__(16) double smem[];
  double* sC = smem;                    // [CH][3][5][15]
  double* sWU = sC + CH * 3 * 75;       // [CH][10]: wq, u
  double* sW = sWU + CH * 10;
  double* sGeo = sW + NN * 5;           // det, invj
  const int tid = threadIdx.x;
  const double gam = g.gamma;
  const int st = tid / NJG, jg = tid % NJG;     // st = s*5 + t
  const bool acc_thread = st < 25;
  const int s_ = st / 5, t_ = st % 5;
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < NN * 5; i += SC::NT) sW[i] = w[(size_t)e * NN * 5 + i];
    if (tid == 0) sGeo[0] = g.det[e];
    if (tid >= 1 && tid < 10) sGeo[tid] = g.invj[(size_t)e * 9 + tid - 1];
    double acc[NN][JG];
#pragma unroll
    for (int i = 0; i < NN; ++i)
#pragma unroll
      for (int jj = 0; jj < JG; ++jj) acc[i][jj] = 0.0;
    for (int c0 = 0; c0 < NPT; c0 += CH) {
      const int npc = min(CH, NPT - c0);
      __syncthreads();
      if (tid < npc) {
        const int pt = c0 + tid;
        double wq[5] = {0, 0, 0, 0, 0}, u[5];
        for (int i = 0; i < NN; ++i) {
          const double a = __ldg(vg.phit + (size_t)i * NPT + pt);
#pragma unroll
          for (int t = 0; t < 5; ++t) wq[t] += a * sW[i * 5 + t];
        }
        to_conservative(wq, g.form, gam, u);
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          sWU[tid * 10 + t] = wq[t];
          sWU[tid * 10 + 5 + t] = u[t];
        }
      }
      __syncthreads();
      for (int item = tid; item < npc * 15; item += SC::NT) {
        const int lp = item / 15, tb = item % 15, pt = c0 + lp;
        double wq[5], u[5];
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          wq[t] = sWU[lp * 10 + t];
          u[t] = sWU[lp * 10 + 5 + t];
        }
        double e1[5][3];
#pragma unroll
        for (int a = 0; a < 5; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) e1[a][b] = (a * 3 + b == tb) ? 1.0 : 0.0;
        double Gv[5][3];
        visc_G(vg, g.form, wq, u, e1, gam, Gv);
        if (pt < NQ) {
          const double vw = g.qw[pt] * sGeo[0];
#pragma unroll
          for (int kk = 0; kk < 3; ++kk) {
            const double j0 = sGeo[1 + kk * 3], j1 = sGeo[2 + kk * 3], j2 = sGeo[3 + kk * 3];
#pragma unroll
            for (int s2 = 0; s2 < 5; ++s2)
              sC[((lp * 3 + kk) * 5 + s2) * 15 + tb] = -(vw * ((j0 * Gv[s2][0] + j1 * Gv[s2][1]) + j2 * Gv[s2][2]));
          }
        } else {
          const int it = pt - NQ, k = it / NQF, qp = it % NQF;
          const double n0 = g.nrm[(size_t)e * 12 + k * 3], n1 = g.nrm[(size_t)e * 12 + k * 3 + 1],
                       n2 = g.nrm[(size_t)e * 12 + k * 3 + 2];
          const double fwq = g.fw[qp] * g.area[(size_t)e * 4 + k];
#pragma unroll
          for (int s2 = 0; s2 < 5; ++s2)
            sC[((lp * 3) * 5 + s2) * 15 + tb] = fwq * ((Gv[s2][0] * n0 + Gv[s2][1] * n1) + Gv[s2][2] * n2);
        }
      }
      __syncthreads();
      if (acc_thread) {
        for (int lp = 0; lp < npc; ++lp) {
          const int pt = c0 + lp;
          // Phi_b[j] for this thread's j pair
          double phi[3][JG];
#pragma unroll
          for (int jj = 0; jj < JG; ++jj) {
            const int j = jg * JG + jj;
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            if (j < NN) {
              t0 = __ldg(vg.tpp + ((size_t)0 * NPT + pt) * NN + j);
              t1 = __ldg(vg.tpp + ((size_t)1 * NPT + pt) * NN + j);
              t2 = __ldg(vg.tpp + ((size_t)2 * NPT + pt) * NN + j);
            }
#pragma unroll
            for (int b = 0; b < 3; ++b) phi[b][jj] = (sGeo[1 + b] * t0 + sGeo[4 + b] * t1) + sGeo[7 + b] * t2;
          }
          const int nkk = pt < NQ ? 3 : 1;
          for (int kk = 0; kk < nkk; ++kk) {
            const double* c = sC + ((lp * 3 + kk) * 5 + s_) * 15 + t_ * 3;
            const double c0v = c[0], c1v = c[1], c2v = c[2];
            double h[JG];
#pragma unroll
            for (int jj = 0; jj < JG; ++jj) h[jj] = (c0v * phi[0][jj] + c1v * phi[1][jj]) + c2v * phi[2][jj];
            const double* tst = pt < NQ ? g.B + ((size_t)pt * 4 + kk) * NN : vg.phipt + (size_t)pt * NN;
#pragma unroll
            for (int i = 0; i < NN; ++i) {
              const double a = __ldg(tst + i);
#pragma unroll
              for (int jj = 0; jj < JG; ++jj) acc[i][jj] += a * h[jj];
            }
          }
        }
      }
    }
    if (acc_thread) {
      double* Se = S + (size_t)e * NM * NM;
#pragma unroll
      for (int i = 0; i < NN; ++i)
#pragma unroll
        for (int jj = 0; jj < JG; ++jj) {
          const int j = jg * JG + jj;
          if (j < NN) Se[(i * 5 + s_) * NM + j * 5 + t_] -= acc[i][jj];
        }
    }
  }
}

}  // namespace mhdg
