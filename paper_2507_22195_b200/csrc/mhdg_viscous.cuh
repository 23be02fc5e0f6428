// Viscous (Navier-Stokes) level-1 condensation on the device (K7).
//
// Reference: macrohdg assembly.py:326-411 (gradient operators, solve_gradient),
// :459-549 (viscous residual terms), :772-976 (viscous linearization,
// S -= A_vq M^-1 A_qv), :1037-1173 (q couplings of the condensed operator);
// gas.py:229-280 (gradient extraction, viscous flux); fluxes.py:222-231.
//
// All per-macro viscous operators are combinations of reference matrices
// with the affine geometry (nothing per macro is stored):
//   M_e^-1        = Mref^-1 / det
//   M_e^-1 K_e,b  = sum_k Jinv[k][b] Pref_k,      Pref_k = Mref^-1 Kref_k
//   K_e,b         = det sum_k Jinv[k][b] Kref_k,   Kref_k[j][i] = sum_q w_q dphi_k[q,j] phi[q,i]
//   E_e,k,b       = area_k n_b Eref_k,             Eref_k[i][j] = sum_q wf_q phi_face_k[q,i] fphi[q,j]
// G(w, q) is linear in q, so dG/dq . y = G(w, y) (exact, no derivative
// tensors are formed or stored).
#pragma once
#include "mhdg_kernels.cuh"

namespace mhdg {

template <int P>
struct ViscDims {
  using D = Dims<P>;
  static constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF, NM = D::NM;
  static constexpr int NQV = NN * 15;   // q per macro
};

// ---------------------------------------------------------------------------
// solve_gradient: q_b = M^-1 (E_b w^ - K_b w)   (assembly.py:398-411)
// ---------------------------------------------------------------------------
template <int P, int NT>
__global__ void __launch_bounds__(NT)
k_solve_gradient(Geo g, ViscGeo vg, const double* __restrict__ w, const double* __restrict__ trace,
                 double* __restrict__ q) {
  using D = Dims<P>;
  constexpr int NN = D::NN, NFN = D::NFN;
  __shared__ double sW[NN * 5], sTR[4 * NFN * 5], sR[NN * 15], sGeo[26];
  __shared__ int sFid[4], sTid[4 * NFN], sRows[4 * NFN];
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * NFN; i += NT) sRows[i] = g.rows[i];
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < NN * 5; i += NT) sW[i] = w[(size_t)e * NN * 5 + i];
    if (tid < 4) sFid[tid] = g.fid[e * 4 + tid];
    for (int i = tid; i < 4 * NFN; i += NT) sTid[i] = g.tidx[(size_t)e * 4 * NFN + i];
    if (tid == 0) sGeo[0] = g.det[e];
    if (tid >= 1 && tid < 10) sGeo[tid] = g.invj[(size_t)e * 9 + tid - 1];
    if (tid >= 10 && tid < 22) sGeo[tid] = g.nrm[(size_t)e * 12 + tid - 10];
    if (tid >= 22 && tid < 26) sGeo[tid] = g.area[(size_t)e * 4 + tid - 22];
    __syncthreads();
    for (int i = tid; i < 4 * NFN * 5; i += NT) {
      const int k = i / (NFN * 5), j = (i / 5) % NFN, s = i % 5;
      sTR[i] = trace[((size_t)sFid[k] * NFN + sTid[k * NFN + j]) * 5 + s];
    }
    __syncthreads();
    // rhs[j][t][b] = -sum_i K_b[j][i] w[i][t] + sum_faces E_k,b tr
    for (int o = tid; o < NN * 15; o += NT) {
      const int j = o / 15, t = (o / 3) % 5, b = o % 3;
      double acc = 0.0;
      for (int k2 = 0; k2 < 3; ++k2) {
        double kk = 0.0;
        for (int i = 0; i < NN; ++i) kk += vg.kref[(k2 * NN + j) * NN + i] * sW[i * 5 + t];
        acc += sGeo[1 + k2 * 3 + b] * kk;
      }
      double r = -(sGeo[0] * acc);
      for (int k = 0; k < 4; ++k)
        for (int jj = 0; jj < NFN; ++jj)
          if (sRows[k * NFN + jj] == j) {
            double ev = 0.0;
            for (int l = 0; l < NFN; ++l) ev += vg.eref[(k * NFN + jj) * NFN + l] * sTR[(k * NFN + l) * 5 + t];
            r += (sGeo[22 + k] * sGeo[10 + k * 3 + b]) * ev;
          }
      sR[o] = r;
    }
    __syncthreads();
    for (int o = tid; o < NN * 15; o += NT) {
      const int i = o / 15, tb = o % 15;
      double acc = 0.0;
      for (int j = 0; j < NN; ++j) acc += vg.minv[i * NN + j] * sR[j * 15 + tb];
      q[(size_t)e * NN * 15 + o] = acc / sGeo[0];
    }
  }
}

// ---------------------------------------------------------------------------
// viscous residual (r_w, r_trace, r_q), CTA per macro, shared-memory
// contractions (assembly.py:459-549 with viscosity)
// ---------------------------------------------------------------------------
template <int P>
struct ResVisc {
  using D = Dims<P>;
  static constexpr int NT = 128;
  static constexpr int GR = 4 * 20 + 1;   // per-q row: kk x (5 r_w + 15 r_q)
  static constexpr size_t bytes = (size_t)(D::NN * 5 + D::NN * 15 + 4 * D::NFN * 5 + D::NQ * GR +
                                           4 * D::NQF * 20 + 4 * D::NQF * 5 + 26) * 8 +
                                  (size_t)(4 * D::NFN * 2 + 4 + 4 * D::NFN + 3 * D::NN) * 4;
};

template <int P>
__global__ void __launch_bounds__(128)
k_residual_visc(Geo g, ViscGeo vg, const double* __restrict__ w, const double* __restrict__ q,
                const double* __restrict__ trace, int has_stage, double alpha, const double* __restrict__ offset,
                int check, double* __restrict__ r_w, double* __restrict__ r_tr, double* __restrict__ r_q,
                unsigned long long* status) {
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF, NT = 128, GR = ResVisc<P>::GR;
  extern __shared__ __align__(16) double smem[];
  double* sW = smem;                     // NN*5
  double* sQ = sW + NN * 5;              // NN*15
  double* sTR = sQ + NN * 15;            // 4*NFN*5
  double* sG = sTR + 4 * NFN * 5;        // NQ*GR
  double* sH = sG + NQ * GR;             // 4*NQF*20: [k][q][ r_w(5) | r_q(15) ]
  double* sHg = sH + 4 * NQF * 20;       // 4*NQF*5 ghost
  double* sGeo = sHg + 4 * NQF * 5;      // 26
  int* sRows = (int*)(sGeo + 26);
  int* sFid = sRows + 4 * NFN;
  int* sTid = sFid + 4;
  int* sNF = sTid + 4 * NFN;
  int* sBnd = sNF + 3 * NN;              // 4 (reuse tail of rows buffer space)
  const int tid = threadIdx.x;
  const double gam = g.gamma;
  for (int i = tid; i < 4 * NFN; i += NT) sRows[i] = g.rows[i];
  for (int i = tid; i < 3 * NN; i += NT) sNF[i] = g.nodef[i];
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < NN * 5; i += NT) sW[i] = w[(size_t)e * NN * 5 + i];
    for (int i = tid; i < NN * 15; i += NT) sQ[i] = q[(size_t)e * NN * 15 + i];
    if (tid < 4) {
      sFid[tid] = g.fid[e * 4 + tid];
      sBnd[tid] = g.bnd ? g.bnd[e * 4 + tid] : 0;
    }
    for (int i = tid; i < 4 * NFN; i += NT) sTid[i] = g.tidx[(size_t)e * 4 * NFN + i];
    if (tid == 0) sGeo[0] = g.det[e];
    if (tid >= 1 && tid < 10) sGeo[tid] = g.invj[(size_t)e * 9 + tid - 1];
    if (tid >= 10 && tid < 22) sGeo[tid] = g.nrm[(size_t)e * 12 + tid - 10];
    if (tid >= 22 && tid < 26) sGeo[tid] = g.area[(size_t)e * 4 + tid - 22];
    __syncthreads();
    for (int i = tid; i < 4 * NFN * 5; i += NT) {
      const int k = i / (NFN * 5), j = (i / 5) % NFN, s = i % 5;
      sTR[i] = trace[((size_t)sFid[k] * NFN + sTid[k * NFN + j]) * 5 + s];
    }
    __syncthreads();
    // volume points: G rows for r_w (F + G) and r_q (mass q, stiffness w)
    for (int qp = tid; qp < NQ; qp += NT) {
      const double* ph = g.B + ((size_t)qp * 4 + 3) * NN;
      double wq[5] = {0, 0, 0, 0, 0}, qq[5][3];
#pragma unroll
      for (int s = 0; s < 5; ++s) qq[s][0] = qq[s][1] = qq[s][2] = 0.0;
      for (int i = 0; i < NN; ++i) {
        const double a = __ldg(ph + i);
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          wq[s] += a * sW[i * 5 + s];
#pragma unroll
          for (int b = 0; b < 3; ++b) qq[s][b] += a * sQ[i * 15 + s * 3 + b];
        }
      }
      double u[5];
      if (!to_conservative(wq, g.form, gam, u)) report(status, 0, 0, e + g.e_base);
      if (check && !admissible(u, gam)) report(status, 0, 2, e + g.e_base);
      double F[5][3], Gv[5][3];
      flux(u, gam, F);
      visc_G(vg, g.form, wq, u, qq, gam, Gv);
      const double vw = g.qw[qp] * sGeo[0];
      double* gr = sG + qp * GR;
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) {
        const double j0 = sGeo[1 + kk * 3], j1 = sGeo[2 + kk * 3], j2 = sGeo[3 + kk * 3];
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          const double f0 = F[s][0] + Gv[s][0], f1 = F[s][1] + Gv[s][1], f2 = F[s][2] + Gv[s][2];
          gr[kk * 20 + s] = -(vw * ((j0 * f0 + j1 * f1) + j2 * f2));
#pragma unroll
          for (int b = 0; b < 3; ++b) gr[kk * 20 + 5 + s * 3 + b] = vw * (sGeo[1 + kk * 3 + b] * wq[s]);
        }
      }
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        double tmp = 0.0;
        if (has_stage) {
          tmp = alpha * u[s];
          if (offset) tmp = tmp + offset[((size_t)e * NQ + qp) * 5 + s];
          tmp = vw * tmp;
        }
        gr[60 + s] = tmp;
#pragma unroll
        for (int b = 0; b < 3; ++b) gr[60 + 5 + s * 3 + b] = vw * qq[s][b];
      }
    }
    // face points: F^ + G^ (viscous normal flux + penalty), r_q face term
    for (int it = tid; it < 4 * NQF; it += NT) {
      const int k = it / NQF, qp = it % NQF;
      const double* pf = g.pf + (size_t)it * NFN;
      const double* fp = g.fphi + (size_t)qp * NFN;
      double wq[5] = {0, 0, 0, 0, 0}, whq[5] = {0, 0, 0, 0, 0}, qq[5][3];
#pragma unroll
      for (int s = 0; s < 5; ++s) qq[s][0] = qq[s][1] = qq[s][2] = 0.0;
      for (int j = 0; j < NFN; ++j) {
        const double a = __ldg(pf + j), b2 = __ldg(fp + j);
        const int row = sRows[k * NFN + j];
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          wq[s] += a * sW[row * 5 + s];
          whq[s] += b2 * sTR[(k * NFN + j) * 5 + s];
#pragma unroll
          for (int b = 0; b < 3; ++b) qq[s][b] += a * sQ[row * 15 + s * 3 + b];
        }
      }
      double u[5], uh[5];
      if (!to_conservative(wq, g.form, gam, u)) report(status, 1 + k, 0, e + g.e_base);
      if (!to_conservative(whq, g.form, gam, uh)) report(status, 1 + k, 1, e + g.e_base);
      if (check && !admissible(u, gam)) report(status, 1 + k, 2, e + g.e_base);
      if (check && !admissible(uh, gam)) report(status, 1 + k, 3, e + g.e_base);
      const double n[3] = {sGeo[10 + k * 3], sGeo[11 + k * 3], sGeo[12 + k * 3]};
      double fh[5], Gv[5][3];
      numerical_flux(g.kind, u, uh, n, gam, fh, g.form == FORM_ENTROPY ? wq : nullptr,
                     g.form == FORM_ENTROPY ? whq : nullptr);
      visc_G(vg, g.form, wq, u, qq, gam, Gv);
      const double fwq = g.fw[qp] * sGeo[22 + k];
      double* h = sH + it * 20;
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const double gn = (Gv[s][0] * n[0] + Gv[s][1] * n[1]) + Gv[s][2] * n[2];
        h[s] = fwq * (fh[s] + (gn - (0.5 * vg.pdiag[s]) * (whq[s] - wq[s])));
#pragma unroll
        for (int b = 0; b < 3; ++b) h[5 + s * 3 + b] = fwq * (whq[s] * n[b]);
      }
      if (sBnd[k] && g.has_uinf) {
        const double mn[3] = {-n[0], -n[1], -n[2]};
        double gh[5], winf[5];
        numerical_flux(g.kind, g.uinf, uh, mn, gam, gh);
        if (g.form == FORM_ENTROPY) entropy_vars(g.uinf, gam, winf);
        else for (int s = 0; s < 5; ++s) winf[s] = g.uinf[s];
#pragma unroll
        for (int s = 0; s < 5; ++s)
          sHg[it * 5 + s] = fwq * (gh[s] + (0.0 - (0.5 * vg.pdiag[s]) * (whq[s] - winf[s])));
      }
    }
    __syncthreads();
    // r_w and r_q: volume contraction + face tests (tile order)
    for (int o = tid; o < NN * 20; o += NT) {
      const int i = o / 20, c = o % 20;
      double av = 0.0, at = 0.0;
      for (int qp = 0; qp < NQ; ++qp) {
        const double* Bq = g.B + (size_t)qp * 4 * NN + i;
        const double* gr = sG + qp * GR + c;
        av += (__ldg(Bq) * gr[0] + __ldg(Bq + NN) * gr[20]) + __ldg(Bq + 2 * NN) * gr[40];
        at += __ldg(Bq + 3 * NN) * gr[60];
      }
      double r = av + at;
      for (int cc = 0; cc < 3; ++cc) {
        const int kj = sNF[i * 3 + cc];
        if (kj < 0) break;
        const int k = kj / NFN, j = kj % NFN;
        double acc = 0.0;
        for (int qp = 0; qp < NQF; ++qp) acc += __ldg(g.pf + (size_t)(k * NQF + qp) * NFN + j) * sH[(k * NQF + qp) * 20 + c];
        r += (c < 5) ? acc : -acc;
      }
      if (c < 5) r_w[((size_t)e * NN + i) * 5 + c] = r;
      else r_q[((size_t)e * NN + i) * 15 + (c - 5)] = r;
    }
    for (int o = tid; o < 4 * NFN * 5; o += NT) {
      const int k = o / (NFN * 5), j = (o / 5) % NFN, s = o % 5;
      double acc = 0.0;
      for (int qp = 0; qp < NQF; ++qp) acc += __ldg(g.fphi + (size_t)qp * NFN + j) * sH[(k * NQF + qp) * 20 + s];
      if (sBnd[k] && g.has_uinf) {
        double ag = 0.0;
        for (int qp = 0; qp < NQF; ++qp) ag += __ldg(g.fphi + (size_t)qp * NFN + j) * sHg[(k * NQF + qp) * 5 + s];
        acc += ag;
      }
      atomicAdd(&r_tr[((size_t)sFid[k] * NFN + sTid[k * NFN + j]) * 5 + s], acc);
    }
  }
}

// ---------------------------------------------------------------------------
// viscous condensed operator pieces (assembly.py:1037-1173), CTA per macro.
//   k_visc_in : g = -r_w[1,2] - vvhat(x)[0,2] + vq(M^-1 (r_q[1,2] + qvhat(x)[0,2]))
//   k_visc_out: y += hh x[0] + hw z - vhatq(M^-1 (qv z + qvhat(x)[0] + r_q[1]))
//   k_visc_dq : d_q = -M^-1 (r_q + qv d_w + qvhat d_trace)
// with qvhat(x)[i][t][b] = -sum_k E_k,b x_k (rows), qv(z) = K_b z, and
// vq / vhatq evaluated matrix-free as G(w_lin, .) at quadrature points.
// ---------------------------------------------------------------------------
// Y (NN x 15) += qvhat(x) : -sum_k (area n_b) Eref_k x_k scattered to rows
template <int P>
__device__ void add_qvhat(const ViscGeo& vg, const double* sGeo, const int* sRows, const double* sX, double* Y,
                          int NT) {
  using D = Dims<P>;
  constexpr int NFN = D::NFN;
  for (int k = 0; k < 4; ++k) {
    for (int o = threadIdx.x; o < NFN * 15; o += NT) {
      const int ip = o / 15, t = (o / 3) % 5, b = o % 3;
      double ev = 0.0;
      for (int j = 0; j < NFN; ++j) ev += vg.eref[(k * NFN + ip) * NFN + j] * sX[(k * NFN + j) * 5 + t];
      Y[sRows[k * NFN + ip] * 15 + t * 3 + b] -= (sGeo[22 + k] * sGeo[10 + k * 3 + b]) * ev;
    }
    __syncthreads();
  }
}

// Y += qv(z) = K_b z
template <int P>
__device__ void add_qv(const ViscGeo& vg, const double* sGeo, const double* sZ, double* Y, int NT) {
  using D = Dims<P>;
  constexpr int NN = D::NN;
  for (int o = threadIdx.x; o < NN * 15; o += NT) {
    const int j = o / 15, t = (o / 3) % 5, b = o % 3;
    double acc = 0.0;
    for (int k2 = 0; k2 < 3; ++k2) {
      double kk = 0.0;
      for (int i = 0; i < NN; ++i) kk += vg.kref[(k2 * NN + j) * NN + i] * sZ[i * 5 + t];
      acc += sGeo[1 + k2 * 3 + b] * kk;
    }
    Y[o] += sGeo[0] * acc;
  }
}

// Yq = M^-1 Y
template <int P>
__device__ void mass_solve(const ViscGeo& vg, const double* sGeo, const double* Y, double* Yq, int NT) {
  using D = Dims<P>;
  constexpr int NN = D::NN;
  for (int o = threadIdx.x; o < NN * 15; o += NT) {
    const int i = o / 15, tb = o % 15;
    double acc = 0.0;
    for (int j = 0; j < NN; ++j) acc += vg.minv[i * NN + j] * Y[j * 15 + tb];
    Yq[o] = acc / sGeo[0];
  }
}

template <int P>
__global__ void __launch_bounds__(128)
k_visc_dq(Geo g, ViscGeo vg, const double* __restrict__ r_q, const double* __restrict__ d_w,
          const double* __restrict__ d_trace, double* __restrict__ d_q) {
  using D = Dims<P>;
  constexpr int NN = D::NN, NFN = D::NFN, NM = D::NM, NT = 128;
  __shared__ double sX[4 * NFN * 5], sY[NN * 15], sYq[NN * 15], sZ[NM], sGeo[26];
  __shared__ int sRows[4 * NFN], sFid[4], sTid[4 * NFN];
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * NFN; i += NT) sRows[i] = g.rows[i];
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < NM; i += NT) sZ[i] = d_w[(size_t)e * NM + i];
    for (int i = tid; i < NN * 15; i += NT) sY[i] = r_q[(size_t)e * NN * 15 + i];
    if (tid < 4) sFid[tid] = g.fid[e * 4 + tid];
    for (int i = tid; i < 4 * NFN; i += NT) sTid[i] = g.tidx[(size_t)e * 4 * NFN + i];
    if (tid == 0) sGeo[0] = g.det[e];
    if (tid >= 1 && tid < 10) sGeo[tid] = g.invj[(size_t)e * 9 + tid - 1];
    if (tid >= 10 && tid < 22) sGeo[tid] = g.nrm[(size_t)e * 12 + tid - 10];
    if (tid >= 22 && tid < 26) sGeo[tid] = g.area[(size_t)e * 4 + tid - 22];
    __syncthreads();
    for (int i = tid; i < 4 * NFN * 5; i += NT) {
      const int k = i / (NFN * 5), j = (i / 5) % NFN, s2 = i % 5;
      sX[i] = d_trace[((size_t)sFid[k] * NFN + sTid[k * NFN + j]) * 5 + s2];
    }
    __syncthreads();
    add_qv<P>(vg, sGeo, sZ, sY, NT);
    __syncthreads();
    add_qvhat<P>(vg, sGeo, sRows, sX, sY, NT);
    mass_solve<P>(vg, sGeo, sY, sYq, NT);
    __syncthreads();
    for (int o = tid; o < NN * 15; o += NT) d_q[(size_t)e * NN * 15 + o] = -sYq[o];
  }
}

// kinetic-energy dissipation partial sums: sum vol_w 0.5 rho |curl V|^2
// (assembly.py:622-648)
template <int P, int NT>
__global__ void __launch_bounds__(NT)
k_dissipation(Geo g, ViscGeo vg, const double* __restrict__ w, const double* __restrict__ q,
              double* __restrict__ partial) {
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ;
  __shared__ double sW[NN * 5], sQ[NN * 15], red[NT];
  double acc = 0.0;
  const double gam = g.gamma;
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < NN * 5; i += NT) sW[i] = w[(size_t)e * NN * 5 + i];
    for (int i = threadIdx.x; i < NN * 15; i += NT) sQ[i] = q[(size_t)e * NN * 15 + i];
    __syncthreads();
    for (int qp = threadIdx.x; qp < NQ; qp += NT) {
      const double* ph = g.B + ((size_t)qp * 4 + 3) * NN;
      double wq[5] = {0, 0, 0, 0, 0}, qq[5][3];
#pragma unroll
      for (int s2 = 0; s2 < 5; ++s2) qq[s2][0] = qq[s2][1] = qq[s2][2] = 0.0;
      for (int i = 0; i < NN; ++i) {
        const double a = __ldg(ph + i);
#pragma unroll
        for (int s2 = 0; s2 < 5; ++s2) {
          wq[s2] += a * sW[i * 5 + s2];
#pragma unroll
          for (int b = 0; b < 3; ++b) qq[s2][b] += a * sQ[i * 15 + s2 * 3 + b];
        }
      }
      double u[5], gv[3][3], gt[3];
      to_conservative(wq, g.form, gam, u);
      vt_grads(g.form, wq, u, qq, gam, gv, gt);
      const double wx = gv[2][1] - gv[1][2], wy = gv[0][2] - gv[2][0], wz = gv[1][0] - gv[0][1];
      const double om2 = (wx * wx + wy * wy) + wz * wz;
      acc += g.qw[qp] * g.det[e] * 0.5 * u[0] * om2;
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int sft = NT / 2; sft > 0; sft >>= 1) {
    if (threadIdx.x < sft) red[threadIdx.x] += red[threadIdx.x + sft];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

}  // namespace mhdg
