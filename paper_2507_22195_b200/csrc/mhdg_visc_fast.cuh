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
  struct In {
    double W[NN * 5], X[4 * NFN * 5], RQ[NN * 15], Gk[NKP * 5], part[WPM][NTI * 8 * 8], geo[26];
    int fid[4], tid[4 * NFN];
  };
  struct Out {
    double W[NN * 5], Z[NM], X[4 * NFN * 5], RQ[NN * 15], Gf[NPF * 5], YQ[NPF * 15], geo[26];
    int fid[4], tid[4 * NFN];
  };
};

template <int P>
MHDG_DEV void vf_load_geo(const Geo& g, int e, double* geo, int* fid, int* tid, int lt, int nt) {
  constexpr int NFN = Dims<P>::NFN;
  for (int i = lt; i < 26 + 4 + 4 * NFN; i += nt) {
    if (i == 0) geo[0] = g.det[e];
    else if (i < 10) geo[i] = g.invj[(size_t)e * 9 + i - 1];
    else if (i < 22) geo[i] = g.nrm[(size_t)e * 12 + i - 10];
    else if (i < 26) geo[i] = g.area[(size_t)e * 4 + i - 22];
    else if (i < 30) fid[i - 26] = g.fid[e * 4 + i - 26];
    else tid[i - 30] = g.tidx[(size_t)e * 4 * NFN + i - 30];
  }
}

// yq contribution of the trace: (area_k n_k,b) sum_jj CX_k[pt][jj] x_k[jj][t]
template <int P>
MHDG_DEV void vf_add_x(const ViscGeo& vg, int pt, const double* X, const double* geo, double yq[5][3]) {
  constexpr int NFN = Dims<P>::NFN, NPT = VFast<P>::NPT;
#pragma unroll 1
  for (int k = 0; k < 4; ++k) {
    double u[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int jj = 0; jj < NFN; ++jj) {
      const double c = __ldg(vg.cxt + (size_t)(k * NFN + jj) * NPT + pt);
#pragma unroll
      for (int t = 0; t < 5; ++t) u[t] += c * X[(k * NFN + jj) * 5 + t];
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
      for (int t = 0; t < 5; ++t) u[t] += c * Z[i * 5 + t];
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
__global__ void __launch_bounds__(128, 4)
k_visc_in2(Geo g, ViscGeo vg, int mode, const double* __restrict__ wlin, const double* __restrict__ hhat,
           const double* __restrict__ x, const double* __restrict__ r_w, const double* __restrict__ r_q,
           double* __restrict__ gout) {
  using V = VFast<P>;
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF, NM = D::NM, NPT = V::NPT;
  constexpr int MB = V::MBI, SP = V::SPI, NK = V::NK;
  extern __shared__ __align__(16) double smem[];
  typename V::In* sm = reinterpret_cast<typename V::In*>(smem);
  const int tid = threadIdx.x, slot = tid / SP, lt = tid % SP;
  const double gam = g.gamma;
  const bool use_x = mode != 1, use_r = mode != 0;
  const int nblk = (g.E + MB - 1) / MB;
  for (int i = NK * 5 + lt; i < V::NKP * 5; i += SP) sm[slot].Gk[i] = 0.0;
  pdl_wait();   // before: shared-memory padding only (mhdg_kernels.cuh PDL invariant)
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int e = blk * MB + slot;
    const bool live = e < g.E;
    typename V::In& S = sm[slot];
    __syncthreads();
    if (live) {
      vf_load_geo<P>(g, e, S.geo, S.fid, S.tid, lt, SP);
      for (int i = lt; i < NN * 5; i += SP) S.W[i] = wlin[(size_t)e * NN * 5 + i];
      if (use_r)
        for (int i = lt; i < NN * 15; i += SP) S.RQ[i] = r_q[(size_t)e * NN * 15 + i];
    }
    __syncthreads();
    if (live && use_x)
      for (int i = lt; i < 4 * NFN * 5; i += SP) {
        const int k = i / (NFN * 5), j = (i / 5) % NFN, s2 = i % 5;
        S.X[i] = x[((size_t)S.fid[k] * NFN + S.tid[k * NFN + j]) * 5 + s2];
      }
    __syncthreads();
    if (live && lt < NPT) {
      const int pt = lt;
      double wq[5] = {0, 0, 0, 0, 0}, yq[5][3];
#pragma unroll
      for (int t = 0; t < 5; ++t) yq[t][0] = yq[t][1] = yq[t][2] = 0.0;
#pragma unroll 4
      for (int i = 0; i < NN; ++i) {
        const double a = __ldg(vg.phit + (size_t)i * NPT + pt);
#pragma unroll
        for (int t = 0; t < 5; ++t) wq[t] += a * S.W[i * 5 + t];
      }
      if (use_x) vf_add_x<P>(vg, pt, S.X, S.geo, yq);
      if (use_r) vf_add_rq<P>(vg, pt, S.RQ, yq);
      const double idet = 1.0 / S.geo[0];
#pragma unroll
      for (int t = 0; t < 5; ++t)
#pragma unroll
        for (int b = 0; b < 3; ++b) yq[t][b] *= idet;
      double u[5], Gv[5][3];
      to_conservative(wq, g.form, gam, u);
      visc_G(vg, g.form, wq, u, yq, gam, Gv);
      if (pt < NQ) {
        const double vw = g.qw[pt] * S.geo[0];
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const double j0 = S.geo[1 + kk * 3], j1 = S.geo[2 + kk * 3], j2 = S.geo[3 + kk * 3];
#pragma unroll
          for (int t = 0; t < 5; ++t)
            S.Gk[(pt * 3 + kk) * 5 + t] = -(vw * ((j0 * Gv[t][0] + j1 * Gv[t][1]) + j2 * Gv[t][2]));
        }
      } else {
        const int it = pt - NQ, k = it / NQF, qp = it % NQF;
        const double fwq = g.fw[qp] * S.geo[22 + k];
        const double n0 = S.geo[10 + k * 3], n1 = S.geo[11 + k * 3], n2 = S.geo[12 + k * 3];
        double hx[5] = {0, 0, 0, 0, 0};
        if (use_x) {
          double xq[5] = {0, 0, 0, 0, 0};
#pragma unroll
          for (int j = 0; j < NFN; ++j) {
            const double b2 = __ldg(g.fphi + qp * NFN + j);
#pragma unroll
            for (int t = 0; t < 5; ++t) xq[t] += b2 * S.X[(k * NFN + j) * 5 + t];
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
    __syncthreads();
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
          dmma_8x8x4(c[nt], a, __ldg(vg.tst + (size_t)K * (NTI * 8) + nt * 8 + (lane >> 2)));
      }
#pragma unroll
      for (int nt = 0; nt < NTI; ++nt) {
        S.part[wl][(nt * 8 + kl * 2) * 8 + sa] = c[nt][0];
        S.part[wl][(nt * 8 + kl * 2 + 1) * 8 + sa] = c[nt][1];
      }
    }
    __syncthreads();
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
__global__ void __launch_bounds__(128)
k_visc_out2(Geo g, ViscGeo vg, int mode, const double* __restrict__ wlin, const double* __restrict__ hh,
            const double* __restrict__ hw, const double* __restrict__ x, const double* __restrict__ z,
            const double* __restrict__ r_q, double* __restrict__ y) {
  using V = VFast<P>;
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF, NM = D::NM;
  constexpr int MB = V::MBO, NPF = V::NPF;
  extern __shared__ __align__(16) double smem[];
  typename V::Out* sm = reinterpret_cast<typename V::Out*>(smem);
  const int tid = threadIdx.x;
  const int slot = tid / NPF, lt = tid % NPF;
  const double gam = g.gamma;
  const int nblk = (g.E + MB - 1) / MB;
  pdl_wait();   // before: index arithmetic only (mhdg_kernels.cuh PDL invariant)
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int e = blk * MB + slot;
    const bool live = slot < MB && e < g.E;
    typename V::Out& S = sm[slot < MB ? slot : 0];
    __syncthreads();
    if (live) {
      vf_load_geo<P>(g, e, S.geo, S.fid, S.tid, lt, NPF);
      for (int i = lt; i < NN * 5; i += NPF) S.W[i] = wlin[(size_t)e * NN * 5 + i];
      for (int i = lt; i < NM; i += NPF) S.Z[i] = z[(size_t)e * NM + i];
      if (mode == 1)
        for (int i = lt; i < NN * 15; i += NPF) S.RQ[i] = r_q[(size_t)e * NN * 15 + i];
    }
    __syncthreads();
    if (live && mode == 0)
      for (int i = lt; i < 4 * NFN * 5; i += NPF) {
        const int k = i / (NFN * 5), j = (i / 5) % NFN, s2 = i % 5;
        S.X[i] = x[((size_t)S.fid[k] * NFN + S.tid[k * NFN + j]) * 5 + s2];
      }
    __syncthreads();
    if (mode == 0) {
      // gradient unknowns at the face points on the FP64 tensor cores, per
      // (macro slot, 8-point tile):
      //   yq = (1/det) sum_k (area n)_k (CX_k x_k) + sum_k2 Jinv[k2] (DZ_k2 z)
      // (the point-per-thread contraction spent one shared-memory load per
      // FMA on the broadcast x / z values)
      constexpr int MT = (NPF + 7) / 8, KX = (NFN + 3) / 4, KZ = (NN + 3) / 4;
      const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, nn = lane >> 2;
      for (int job = warp; job < MB * MT; job += V::NT / 32) {
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
            const double b = (jj < NFN && nn < 5) ? Sx.X[(k * NFN + jj) * 5 + nn] : 0.0;
            dmma_8x8x4(c, __ldg(vg.cxf + ((k * MT + mt) * KX + ks) * 32 + lane), b);
          }
          const double a = Sx.geo[22 + k];
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const double an = a * Sx.geo[10 + k * 3 + b];
            acc[0][b] += an * c[0];
            acc[1][b] += an * c[1];
          }
        }
        const double idet = 1.0 / Sx.geo[0];
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
            const double b = (i < NN && nn < 5) ? Sx.Z[i * 5 + nn] : 0.0;
            dmma_8x8x4(c, __ldg(vg.dzf + ((k2 * MT + mt) * KZ + ks) * 32 + lane), b);
          }
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const double jb = Sx.geo[1 + k2 * 3 + b];
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
      __syncthreads();
    }
    if (live) {
      const int it = lt, k = it / NQF, qp = it % NQF, pt = NQ + it;
      double wq[5] = {0, 0, 0, 0, 0}, zq[5] = {0, 0, 0, 0, 0}, xq[5] = {0, 0, 0, 0, 0}, yq[5][3];
#pragma unroll
      for (int t = 0; t < 5; ++t) yq[t][0] = yq[t][1] = yq[t][2] = 0.0;
#pragma unroll
      for (int j = 0; j < NFN; ++j) {
        const double a = __ldg(g.pf + (size_t)it * NFN + j);
        const int row = __ldg(g.rows + k * NFN + j);
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          wq[t] += a * S.W[row * 5 + t];
          zq[t] += a * S.Z[row * 5 + t];
        }
        if (mode == 0) {
          const double b2 = __ldg(g.fphi + qp * NFN + j);
#pragma unroll
          for (int t = 0; t < 5; ++t) xq[t] += b2 * S.X[(k * NFN + j) * 5 + t];
        }
      }
      if (mode == 0) {
#pragma unroll
        for (int t = 0; t < 5; ++t)
#pragma unroll
          for (int b = 0; b < 3; ++b) yq[t][b] = S.YQ[it * 15 + t * 3 + b];
      } else {
        if (mode == 1) vf_add_rq<P>(vg, pt, S.RQ, yq);
        const double idet = 1.0 / S.geo[0];
#pragma unroll
        for (int t = 0; t < 5; ++t)
#pragma unroll
          for (int b = 0; b < 3; ++b) yq[t][b] *= idet;
        vf_add_z<P>(vg, pt, S.Z, S.geo, yq);
      }
      double u[5], Gv[5][3];
      to_conservative(wq, g.form, gam, u);
      visc_G(vg, g.form, wq, u, yq, gam, Gv);
      const double fwq = g.fw[qp] * S.geo[22 + k];
      const double n0 = S.geo[10 + k * 3], n1 = S.geo[11 + k * 3], n2 = S.geo[12 + k * 3];
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
    __syncthreads();
    // trace tests on DMMA, per (macro slot, face): C[j][s] = sum_qp fphi[qp][j] Gf[qp][s]
    // (A fragments of fphi from the fragment-ordered table vg.fpf)
    {
      constexpr int TM = (NFN + 7) / 8, TK = (NQF + 3) / 4;
      const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, nn = lane >> 2;
      for (int job = warp; job < MB * 4; job += V::NT / 32) {
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
          for (int t = 0; t < TM; ++t) dmma_8x8x4(c[t], __ldg(vg.fpf + (t * TK + ks) * 32 + lane), b);
        }
#pragma unroll
        for (int t = 0; t < TM; ++t)
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int j = t * 8 + nn, s2 = kq * 2 + h2;
            if (j < NFN && s2 < 5)
              atomicAdd(&y[((size_t)Sx.fid[k] * NFN + Sx.tid[k * NFN + j]) * 5 + s2], c[t][h2]);
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
