// Viscous flux algebra (gas.py:229-280), templated like mhdg_math.cuh.
#pragma once
#include "mhdg_math.cuh"

namespace mhdg {

struct ViscGeo {
  double mu_eff, kappa;
  double pdiag[5];                 // penalty diagonal (fluxes.py:222-231)
  const double* minv;              // (NN, NN)   Mref^-1
  const double* pref;              // (3, NN, NN) Mref^-1 Kref_k
  const double* kref;              // (3, NN, NN) Kref_k[j][i]
  const double* eref;              // (4, NFN, NFN) Eref_k[i][j]
  // point tables (built at context creation; pt = NQ volume points, then the
  // 4 NQF face points k*NQF+qf; phi_pt is dense over the NN macro nodes)
  int npt;
  const double* phit;              // (NN, NPT)   phi_pt^T
  const double* phipt;             // (NPT, NN)   phi_pt
  const double* pmt;               // (NN, NPT)   (phi_pt Mref^-1)^T
  const double* cxt;               // (4, NFN, NPT)  -(phi_pt Mref^-1 R_k Eref_k)^T
  const double* dzt;               // (3, NN, NPT)   (phi_pt Mref^-1 Kref_k)^T
  const double* tpp;               // (3, NPT, NN)   phi_pt Pref_k
  const double* tst;               // (NKP, NTI*8)   test rows: dphi_kk at (q,kk), then phi_pt at face pts
  // face-point slices of cxt / dzt as lane-swizzled DMMA A fragments:
  // cxf [k][mt][ks][lane] = cxt[k][jj = 4 ks + lane % 4][NQ + 8 mt + lane / 4]
  // dzf [k2][mt][ks][lane] = dzt[k2][i = 4 ks + lane % 4][NQ + 8 mt + lane / 4]
  const double* cxf;
  const double* dzf;
  const double* fpf;               // fphi as A fragments [mt][ks][lane] = fphi[q = 4 ks + lane % 4][j = 8 mt + lane / 4]
};

// velocity / temperature gradients from the working variables (gas.py:229-262)
template <class T, class Q>
MHDG_DEV void vt_grads(int form, const T w[5], const T u[5], const Q g[5][3], double gam, T gv[3][3],
                       T gt[3]) {
  if (form == FORM_ENTROPY) {
    const T ve = w[4];
    const T ive2 = dv(1.0, ve * ve);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) gv[i][j] = (w[1 + i] * g[4][j] - ve * g[1 + i][j]) * ive2;
#pragma unroll
    for (int j = 0; j < 3; ++j) gt[j] = (gam * g[4][j]) * ive2;
    return;
  }
  T rho, vel[3], p;
  primitive(u, gam, rho, vel, p);
  const T irho = dv(1.0, rho);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) gv[i][j] = (g[1 + i][j] - vel[i] * g[0][j]) * irho;
  const T ke = 0.5 * ((vel[0] * vel[0] + vel[1] * vel[1]) + vel[2] * vel[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const T conv = (u[1] * gv[0][j] + u[2] * gv[1][j]) + u[3] * gv[2][j];
    const T gp = (gam - 1.0) * (g[4][j] - ke * g[0][j] - conv);
    gt[j] = gam * (rho * gp - p * g[0][j]) * (irho * irho);
  }
}

// diffusive flux tensor G[s][a] (gas.py:264-280); vel from the conservative state
template <class T>
MHDG_DEV void viscous_flux(const ViscGeo& vg, const T vel[3], const T gv[3][3], const T gt[3], T G[5][3]) {
  const T div = (gv[0][0] + gv[1][1]) + gv[2][2];
  T tau[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) tau[i][j] = vg.mu_eff * (gv[i][j] + gv[j][i]);
#pragma unroll
  for (int i = 0; i < 3; ++i) tau[i][i] = tau[i][i] - (2.0 / 3.0) * vg.mu_eff * div;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    G[0][j] = from_d<T>(0.0);
#pragma unroll
    for (int i = 0; i < 3; ++i) G[1 + i][j] = -tau[i][j];
    G[4][j] = -(((tau[0][j] * vel[0] + tau[1][j] * vel[1]) + tau[2][j] * vel[2]) + vg.kappa * gt[j]);
  }
}

// G(w, q) at one point: w working variables, u = u(w), q gradient (5 x 3)
template <class T, class Q>
MHDG_DEV void visc_G(const ViscGeo& vg, int form, const T w[5], const T u[5], const Q q[5][3], double gam,
                     T G[5][3]) {
  T gv[3][3], gt[3];
  vt_grads(form, w, u, q, gam, gv, gt);
  T rho, vel[3], p;
  primitive(u, gam, rho, vel, p);
  viscous_flux(vg, vel, gv, gt, G);
}

}  // namespace mhdg
