// mhdg_macro.cuh -- the operator for m > 1 macro subdivision.
//
// With m > 1 a macro-tetrahedron holds n_sub = m^3 Kuhn sub-elements that
// share a C0 node space (nc nodes per macro), and each macro face carries
// n_st / 4 = m^2 side tiles whose facet nodes map into a C0 trace space of
// nt nodes per face (reference fem.py:550-724, assembly.py:155-324).  The
// kernels here are the generic forms of K1-K6 for that layout, one CTA per
// macro (persistent grid), templated on the element degree P only:
//   mm_residual      assembly.py:459-549 (volume per sub-element, face per tile)
//   mm_linearize     assembly.py:772-976: S assembled in global memory
//                    (dual-number Jacobians), inverted by the batched
//                    Gauss-Jordan kernels of mhdg_gj_blocked.cuh
//   mm_face_in/out   the condensed operator's tile couplings (assembly.py:
//                    1086-1143) around the per-macro S^-1 GEMV
//   mm_precond_blk   face blocks (assembly.py:994-1026) from the face's tiles
// Trace-space sums (r_trace, y, b, face blocks) are deterministic: tile
// contributions go to a per-(macro, tile, facet node) buffer and each trace
// node gathers its contributions through a CSR list in the reference's
// np.add.at order (tile, then macro, then node), so results are bitwise
// reproducible run to run (reference test_assembly.py:109-115).
// Inviscid, periodic meshes; the m = 1 path keeps its specialised kernels.
#pragma once

namespace mhdg {

struct MGeo {
  int E, F, nsub, nst, nc, nt;
  int form, kind;
  double gamma;
  const double* phi;     // (NQ, NN)
  const double* dphi;    // (NQ, NN, 3)
  const double* qw;      // (NQ)
  const double* pf;      // (nst, NQF, NFN) phi_face per tile
  const double* fphi;    // (NQF, NFN)
  const double* fw;      // (NQF)
  const int* scatter;    // (nsub, NN) element node -> macro C0 node
  const int* rows;       // (nst, NFN) facet node -> macro C0 node
  const double* det;     // (E, nsub)
  const double* invj;    // (E, nsub, 9)
  const double* nrm;     // (E, nst, 3)
  const double* area;    // (E, nst) area * (d-1)!
  const int* fid;        // (E, nst)
  const int* tidx;       // (E, nst, NFN)
  const int* tptr;       // (F * nt + 1) CSR over trace entries
  const int* tlist;      // contribution slots (e * nst + k) * NFN + j
  const int* fptr;       // (F + 1) tiles of each face
  const int* flist;      // tile ids e * nst + k
};

// status key of the m > 1 kernels: ((loc * 4 + sub) << 40) | macro with
// loc = sub-element s (volume) or nsub + k (tile k): the smallest key is the
// reference's first failure in loop order (volume subs, then tiles)
__device__ __forceinline__ void mm_report(unsigned long long* st, int loc, int sub, long long item) {
  atomicMin(st, ((unsigned long long)(loc * 4 + sub) << 40) | (unsigned long long)item);
}

// ---------------------------------------------------------------------------
// residual: r_w per macro in shared memory, tile contributions to r_trace in
// the contribution buffer cb (gathered by mm_gather)
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(128)
mm_residual(MGeo g, const double* __restrict__ w, const double* __restrict__ tr, int has_stage, double alpha,
            const double* __restrict__ offset, int check, double* __restrict__ r_w, double* __restrict__ cb,
            unsigned long long* status) {
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF;
  extern __shared__ __align__(16) double sm[];
  const int NC = g.nc;
  double* sW = sm;                  // NC*5
  double* sR = sW + NC * 5;         // NC*5
  double* sG = sR + NC * 5;         // NQ*20 (volume) / NQF*5 (faces)
  const double gam = g.gamma;
  const int tid = threadIdx.x;
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < NC * 5; i += 128) {
      sW[i] = w[(size_t)e * NC * 5 + i];
      sR[i] = 0.0;
    }
    __syncthreads();
    for (int s = 0; s < g.nsub; ++s) {
      const int* sc = g.scatter + s * NN;
      const double det = g.det[(size_t)e * g.nsub + s];
      const double* ij = g.invj + ((size_t)e * g.nsub + s) * 9;
      for (int q = tid; q < NQ; q += 128) {
        double wq[5] = {0, 0, 0, 0, 0};
        for (int i = 0; i < NN; ++i) {
          const double a = g.phi[q * NN + i];
          const double* wi = sW + sc[i] * 5;
#pragma unroll
          for (int c = 0; c < 5; ++c) wq[c] += a * wi[c];
        }
        double u[5];
        if (!to_conservative(wq, g.form, gam, u)) mm_report(status, s, 0, e);
        if (check && !admissible(u, gam)) mm_report(status, s, 2, e);
        double F[5][3];
        flux(u, gam, F);
        const double vw = g.qw[q] * det;
        double* gr = sG + q * 20;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk)
#pragma unroll
          for (int c = 0; c < 5; ++c)
            gr[kk * 5 + c] = -(vw * ((ij[kk * 3 + 0] * F[c][0] + ij[kk * 3 + 1] * F[c][1]) + ij[kk * 3 + 2] * F[c][2]));
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double t = 0.0;
          if (has_stage) {
            t = alpha * u[c];
            if (offset) t = t + offset[(((size_t)e * g.nsub + s) * NQ + q) * 5 + c];
            t = vw * t;
          }
          gr[15 + c] = t;
        }
      }
      __syncthreads();
      for (int o = tid; o < NN * 5; o += 128) {
        const int i = o / 5, c = o % 5;
        double acc = 0.0;
        for (int q = 0; q < NQ; ++q) {
          const double* gr = sG + q * 20;
          const double* dp = g.dphi + ((size_t)q * NN + i) * 3;
          acc += ((dp[0] * gr[c] + dp[1] * gr[5 + c]) + dp[2] * gr[10 + c]) + g.phi[q * NN + i] * gr[15 + c];
        }
        sR[sc[i] * 5 + c] += acc;
      }
      __syncthreads();
    }
    for (int k = 0; k < g.nst; ++k) {
      const int* rows = g.rows + k * NFN;
      const int f = g.fid[(size_t)e * g.nst + k];
      const int* td = g.tidx + ((size_t)e * g.nst + k) * NFN;
      const double* pfk = g.pf + (size_t)k * NQF * NFN;
      const double ar = g.area[(size_t)e * g.nst + k];
      const double* nr = g.nrm + ((size_t)e * g.nst + k) * 3;
      for (int q = tid; q < NQF; q += 128) {
        double wq[5] = {0, 0, 0, 0, 0}, wh[5] = {0, 0, 0, 0, 0};
        for (int j = 0; j < NFN; ++j) {
          const double a = pfk[q * NFN + j], b = g.fphi[q * NFN + j];
          const double* wj = sW + rows[j] * 5;
          const double* tj = tr + ((size_t)f * g.nt + td[j]) * 5;
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            wq[c] += a * wj[c];
            wh[c] += b * tj[c];
          }
        }
        double u[5], uh[5];
        if (!to_conservative(wq, g.form, gam, u)) mm_report(status, g.nsub + k, 0, e);
        if (!to_conservative(wh, g.form, gam, uh)) mm_report(status, g.nsub + k, 1, e);
        if (check && !admissible(u, gam)) mm_report(status, g.nsub + k, 2, e);
        if (check && !admissible(uh, gam)) mm_report(status, g.nsub + k, 3, e);
        const double n[3] = {nr[0], nr[1], nr[2]};
        double fh[5];
        numerical_flux(g.kind, u, uh, n, gam, fh, g.form == FORM_ENTROPY ? wq : nullptr,
                       g.form == FORM_ENTROPY ? wh : nullptr);
        const double fwq = g.fw[q] * ar;
#pragma unroll
        for (int c = 0; c < 5; ++c) sG[q * 5 + c] = fwq * fh[c];
      }
      __syncthreads();
      for (int o = tid; o < 2 * NFN * 5; o += 128) {
        const int half = o / (NFN * 5), j = (o / 5) % NFN, c = o % 5;
        double acc = 0.0;
        if (half == 0) {
          for (int q = 0; q < NQF; ++q) acc += pfk[q * NFN + j] * sG[q * 5 + c];
          sR[rows[j] * 5 + c] += acc;
        } else {
          for (int q = 0; q < NQF; ++q) acc += g.fphi[q * NFN + j] * sG[q * 5 + c];
          cb[(((size_t)e * g.nst + k) * NFN + j) * 5 + c] = acc;
        }
      }
      __syncthreads();
    }
    for (int i = tid; i < NC * 5; i += 128) r_w[(size_t)e * NC * 5 + i] = sR[i];
  }
}

// out[t] (+)= sum of the contributions listed for trace entry t, in list
// order; mode 0: out = sum, 1: out = a[t] - sum, 2: out = -a[t] - sum
__global__ void mm_gather(int n_entries, const int* __restrict__ ptr, const int* __restrict__ list,
                          const double* __restrict__ cb, int mode, const double* __restrict__ a,
                          double* __restrict__ out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_entries * 5; t += gridDim.x * blockDim.x) {
    const int ent = t / 5, c = t % 5;
    double acc = 0.0;
    for (int l = ptr[ent]; l < ptr[ent + 1]; ++l) acc += cb[(size_t)list[l] * 5 + c];
    out[t] = mode == 0 ? acc : (mode == 1 ? a[t] - acc : (-a[t]) - acc);
  }
}

// volume states u at the quadrature points of every sub-element: (E, nsub, NQ, 5)
template <int P>
__global__ void mm_volume_states(MGeo g, const double* __restrict__ w, double* __restrict__ out,
                                 unsigned long long* status) {
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ;
  const int64_t n = (int64_t)g.E * g.nsub * NQ;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(t % NQ), s = (int)((t / NQ) % g.nsub);
    const int64_t e = t / ((int64_t)NQ * g.nsub);
    double wq[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < NN; ++i) {
      const double a = g.phi[q * NN + i];
      const double* wi = w + ((size_t)e * g.nc + g.scatter[s * NN + i]) * 5;
#pragma unroll
      for (int c = 0; c < 5; ++c) wq[c] += a * wi[c];
    }
    double u[5];
    if (!to_conservative(wq, g.form, g.gamma, u)) mm_report(status, s, 0, e);
#pragma unroll
    for (int c = 0; c < 5; ++c) out[t * 5 + c] = u[c];
  }
}

// five volume integrals (assembly.py:595-620), per-block partial sums
template <int P>
__global__ void __launch_bounds__(128) mm_integrals(MGeo g, const double* __restrict__ w, double* __restrict__ part) {
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ;
  __shared__ double red[5][128];
  double acc[5] = {0, 0, 0, 0, 0};
  const double gam = g.gamma;
  const int64_t n = (int64_t)g.E * g.nsub * NQ;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(t % NQ), s = (int)((t / NQ) % g.nsub);
    const int64_t e = t / ((int64_t)NQ * g.nsub);
    double wq[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < NN; ++i) {
      const double a = g.phi[q * NN + i];
      const double* wi = w + ((size_t)e * g.nc + g.scatter[s * NN + i]) * 5;
#pragma unroll
      for (int c = 0; c < 5; ++c) wq[c] += a * wi[c];
    }
    double u[5];
    to_conservative(wq, g.form, gam, u);
    double rho, vel[3], p;
    primitive(u, gam, rho, vel, p);
    const double vw = g.qw[q] * g.det[(size_t)e * g.nsub + s];
    const double sp = ::log(p) - gam * ::log(rho);
    acc[0] += vw * (-rho * sp / (gam - 1.0));
    acc[1] += vw * rho * sp;
    acc[2] += vw * 0.5 * rho * ((vel[0] * vel[0] + vel[1] * vel[1]) + vel[2] * vel[2]);
    acc[3] += vw * rho;
    acc[4] += vw * u[4];
  }
  for (int c = 0; c < 5; ++c) red[c][threadIdx.x] = acc[c];
  __syncthreads();
  for (int sft = 64; sft > 0; sft >>= 1) {
    if (threadIdx.x < sft)
      for (int c = 0; c < 5; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + sft];
    __syncthreads();
  }
  if (threadIdx.x < 5) part[blockIdx.x * 5 + threadIdx.x] = red[threadIdx.x][0];
}

// ---------------------------------------------------------------------------
// linearization: S (row-major, (i s) x (j t)) per macro in `sm_` (global),
// face tensors hw / hhat / hh as (E, nst, NQF, 5, 5) [s][t]
// ---------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(128)
mm_linearize(MGeo g, const double* __restrict__ w, const double* __restrict__ tr, double weight, double ptc,
             double* __restrict__ S, double* __restrict__ hw_out, double* __restrict__ hhat_out,
             double* __restrict__ hh_out) {
  using D = Dims<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF;
  extern __shared__ __align__(16) double sm[];
  const int NC = g.nc, NM = 5 * NC;
  double* sW = sm;               // NC*5
  double* sC = sW + NC * 5;      // NQ * 4 * 25: [q][kk][s*5+t] (kk = 3: temporal)
  const double gam = g.gamma;
  const int tid = threadIdx.x;
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    double* Se = S + (size_t)e * NM * NM;
    __syncthreads();
    for (int i = tid; i < NC * 5; i += 128) sW[i] = w[(size_t)e * NC * 5 + i];
    for (size_t i = tid; i < (size_t)NM * NM; i += 128) Se[i] = 0.0;
    __syncthreads();
    for (int s = 0; s < g.nsub; ++s) {
      const int* sc = g.scatter + s * NN;
      const double det = g.det[(size_t)e * g.nsub + s];
      const double* ij = g.invj + ((size_t)e * g.nsub + s) * 9;
      for (int it = tid; it < NQ * 5; it += 128) {
        const int q = it / 5, t = it % 5;
        double wq[5] = {0, 0, 0, 0, 0};
        for (int i = 0; i < NN; ++i) {
          const double a = g.phi[q * NN + i];
          const double* wi = sW + sc[i] * 5;
#pragma unroll
          for (int c = 0; c < 5; ++c) wq[c] += a * wi[c];
        }
        Dual wd[5], ud[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) wd[c] = mk(wq[c], c == t ? 1.0 : 0.0);
        to_conservative(wd, g.form, gam, ud);
        Dual F[5][3];
        flux(ud, gam, F);
        const double vw = g.qw[q] * det;
        double* C = sC + (size_t)q * 100;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk)
#pragma unroll
          for (int c = 0; c < 5; ++c)
            C[kk * 25 + c * 5 + t] = -(vw * ((ij[kk * 3 + 0] * F[c][0].d + ij[kk * 3 + 1] * F[c][1].d) +
                                              ij[kk * 3 + 2] * F[c][2].d));
#pragma unroll
        for (int c = 0; c < 5; ++c) C[75 + c * 5 + t] = weight * (vw * ud[c].d);
      }
      __syncthreads();
      // block[i s][j t] = sum_q (sum_kk dphi_i,kk C[kk][st] + phi_i C[3][st]) phi_j
      for (int ijp = tid; ijp < NN * NN; ijp += 128) {
        const int i = ijp / NN, j = ijp % NN;
        double acc[25];
#pragma unroll
        for (int st = 0; st < 25; ++st) acc[st] = 0.0;
        for (int q = 0; q < NQ; ++q) {
          const double* dp = g.dphi + ((size_t)q * NN + i) * 3;
          const double d0 = dp[0], d1 = dp[1], d2 = dp[2], pi = g.phi[q * NN + i], pj = g.phi[q * NN + j];
          const double* C = sC + (size_t)q * 100;
#pragma unroll
          for (int st = 0; st < 25; ++st)
            acc[st] += (((d0 * C[st] + d1 * C[25 + st]) + d2 * C[50 + st]) + pi * C[75 + st]) * pj;
        }
        const int ri = sc[i] * 5, cj = sc[j] * 5;
#pragma unroll
        for (int st = 0; st < 25; ++st) Se[(size_t)(ri + st / 5) * NM + cj + st % 5] += acc[st];
      }
      __syncthreads();
    }
    for (int k = 0; k < g.nst; ++k) {
      const int* rows = g.rows + k * NFN;
      const int f = g.fid[(size_t)e * g.nst + k];
      const int* td = g.tidx + ((size_t)e * g.nst + k) * NFN;
      const double* pfk = g.pf + (size_t)k * NQF * NFN;
      const double ar = g.area[(size_t)e * g.nst + k];
      const double* nr = g.nrm + ((size_t)e * g.nst + k) * 3;
      const size_t tb = ((size_t)e * g.nst + k) * NQF * 25;
      for (int it = tid; it < NQF * 10; it += 128) {
        const int q = it / 10, t = (it % 10) % 5, which = (it % 10) / 5;
        double wq[5] = {0, 0, 0, 0, 0}, wh[5] = {0, 0, 0, 0, 0};
        for (int j = 0; j < NFN; ++j) {
          const double a = pfk[q * NFN + j], b = g.fphi[q * NFN + j];
          const double* wj = sW + rows[j] * 5;
          const double* tj = tr + ((size_t)f * g.nt + td[j]) * 5;
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            wq[c] += a * wj[c];
            wh[c] += b * tj[c];
          }
        }
        Dual wd[5], whd[5], ud[5], uhd[5], fd[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          wd[c] = mk(wq[c], (which == 0 && c == t) ? 1.0 : 0.0);
          whd[c] = mk(wh[c], (which == 1 && c == t) ? 1.0 : 0.0);
        }
        to_conservative(wd, g.form, gam, ud);
        to_conservative(whd, g.form, gam, uhd);
        const double n[3] = {nr[0], nr[1], nr[2]};
        numerical_flux(g.kind, ud, uhd, n, gam, fd, g.form == FORM_ENTROPY ? wd : nullptr,
                       g.form == FORM_ENTROPY ? whd : nullptr);
        double* dst = (which == 0 ? hw_out : hhat_out) + tb + q * 25;
#pragma unroll
        for (int c = 0; c < 5; ++c) dst[c * 5 + t] = fd[c].d;
        if (which == 1) {
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            double v = fd[c].d;
            if (ptc != 0.0) v = v + (-ptc * uhd[c].d);
            hh_out[tb + q * 25 + c * 5 + t] = v;
          }
        }
      }
      __syncthreads();
      // S face block: sum_q face_w phi_face_i hw[s][t] phi_face_j
      for (int ijp = tid; ijp < NFN * NFN; ijp += 128) {
        const int i = ijp / NFN, j = ijp % NFN;
        double acc[25];
#pragma unroll
        for (int st = 0; st < 25; ++st) acc[st] = 0.0;
        for (int q = 0; q < NQF; ++q) {
          const double ci = (g.fw[q] * ar) * pfk[q * NFN + i], pj = pfk[q * NFN + j];
          const double* h = hw_out + tb + q * 25;
#pragma unroll
          for (int st = 0; st < 25; ++st) acc[st] += (ci * h[st]) * pj;
        }
        const int ri = rows[i] * 5, cj = rows[j] * 5;
#pragma unroll
        for (int st = 0; st < 25; ++st) Se[(size_t)(ri + st / 5) * NM + cj + st % 5] += acc[st];
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// condensed operator pieces
// ---------------------------------------------------------------------------
// local right-hand side per macro: g = sign_r * r (if r) - apply_vvhat(x) (if x)
//   apply_vvhat(x)[rows_k] += sum_q face_w phi_face hhat (fphi x_k)
template <int P>
__global__ void __launch_bounds__(128)
mm_face_in(MGeo g, const double* __restrict__ hhat, const double* __restrict__ x, const double* __restrict__ r,
           double sign_r, double* __restrict__ gout) {
  using D = Dims<P>;
  constexpr int NFN = D::NFN, NQF = D::NQF;
  extern __shared__ __align__(16) double sm[];
  const int NC = g.nc;
  double* sA = sm;              // NC*5 accumulator
  double* sT = sA + NC * 5;     // NQF*5
  const int tid = threadIdx.x;
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < NC * 5; i += 128) sA[i] = 0.0;
    __syncthreads();
    if (x) {
      for (int k = 0; k < g.nst; ++k) {
        const int* rows = g.rows + k * NFN;
        const int f = g.fid[(size_t)e * g.nst + k];
        const int* td = g.tidx + ((size_t)e * g.nst + k) * NFN;
        const double* pfk = g.pf + (size_t)k * NQF * NFN;
        const double ar = g.area[(size_t)e * g.nst + k];
        const size_t tb = ((size_t)e * g.nst + k) * NQF * 25;
        for (int q = tid; q < NQF; q += 128) {
          double xq[5] = {0, 0, 0, 0, 0};
          for (int j = 0; j < NFN; ++j) {
            const double b = g.fphi[q * NFN + j];
            const double* xj = x + ((size_t)f * g.nt + td[j]) * 5;
#pragma unroll
            for (int c = 0; c < 5; ++c) xq[c] += b * xj[c];
          }
          const double* h = hhat + tb + q * 25;
          const double fwq = g.fw[q] * ar;
#pragma unroll
          for (int c = 0; c < 5; ++c) {
            double v = 0.0;
#pragma unroll
            for (int t = 0; t < 5; ++t) v += h[c * 5 + t] * xq[t];
            sT[q * 5 + c] = fwq * v;
          }
        }
        __syncthreads();
        for (int o = tid; o < NFN * 5; o += 128) {
          const int j = o / 5, c = o % 5;
          double acc = 0.0;
          for (int q = 0; q < NQF; ++q) acc += pfk[q * NFN + j] * sT[q * 5 + c];
          sA[rows[j] * 5 + c] += acc;
        }
        __syncthreads();
      }
    }
    for (int i = tid; i < NC * 5; i += 128) {
      double v = -sA[i];
      if (r) v = sign_r * r[(size_t)e * NC * 5 + i] + v;
      gout[(size_t)e * NC * 5 + i] = v;
    }
  }
}

// tile contributions to the trace: cb[(e,k,j),c] = sum_q face_w fphi_j
//   (hh (fphi x_k) [if x] + hw (phi_face z_k) [if z])
template <int P>
__global__ void __launch_bounds__(128)
mm_face_out(MGeo g, const double* __restrict__ hh, const double* __restrict__ hw, const double* __restrict__ x,
            const double* __restrict__ z, double* __restrict__ cb) {
  using D = Dims<P>;
  constexpr int NFN = D::NFN, NQF = D::NQF;
  __shared__ double sT[NQF * 5];
  const int NC = g.nc;
  const int tid = threadIdx.x;
  for (int ek = blockIdx.x; ek < g.E * g.nst; ek += gridDim.x) {
    const int e = ek / g.nst, k = ek % g.nst;
    const int* rows = g.rows + k * NFN;
    const int f = g.fid[ek];
    const int* td = g.tidx + (size_t)ek * NFN;
    const double* pfk = g.pf + (size_t)k * NQF * NFN;
    const double ar = g.area[ek];
    const size_t tb = (size_t)ek * NQF * 25;
    __syncthreads();
    for (int q = tid; q < NQF; q += 128) {
      double v[5] = {0, 0, 0, 0, 0};
      if (x) {
        double xq[5] = {0, 0, 0, 0, 0};
        for (int j = 0; j < NFN; ++j) {
          const double b = g.fphi[q * NFN + j];
          const double* xj = x + ((size_t)f * g.nt + td[j]) * 5;
#pragma unroll
          for (int c = 0; c < 5; ++c) xq[c] += b * xj[c];
        }
        const double* h = hh + tb + q * 25;
#pragma unroll
        for (int c = 0; c < 5; ++c)
#pragma unroll
          for (int t = 0; t < 5; ++t) v[c] += h[c * 5 + t] * xq[t];
      }
      if (z) {
        double zq[5] = {0, 0, 0, 0, 0};
        for (int j = 0; j < NFN; ++j) {
          const double a = pfk[q * NFN + j];
          const double* zj = z + ((size_t)e * NC + rows[j]) * 5;
#pragma unroll
          for (int c = 0; c < 5; ++c) zq[c] += a * zj[c];
        }
        const double* h = hw + tb + q * 25;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          double a2 = 0.0;
#pragma unroll
          for (int t = 0; t < 5; ++t) a2 += h[c * 5 + t] * zq[t];
          v[c] = v[c] + a2;
        }
      }
      const double fwq = g.fw[q] * ar;
#pragma unroll
      for (int c = 0; c < 5; ++c) sT[q * 5 + c] = fwq * v[c];
    }
    __syncthreads();
    for (int o = tid; o < NFN * 5; o += 128) {
      const int j = o / 5, c = o % 5;
      double acc = 0.0;
      for (int q = 0; q < NQF; ++q) acc += g.fphi[q * NFN + j] * sT[q * 5 + c];
      cb[((size_t)ek * NFN + j) * 5 + c] = acc;
    }
  }
}

// y_m = A_m x_m for nmat column-major N x N matrices (S^-1, face-block
// inverses): one row per thread (blockDim >= N), four independent
// accumulators over the columns so each thread keeps four streaming loads in
// flight; the columns' loads are coalesced across the rows.
__global__ void __launch_bounds__(512)
mm_gemv(int nmat, int N, const double* __restrict__ A, const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(16) double sx[];
  for (int m = blockIdx.x; m < nmat; m += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) sx[i] = x[(size_t)m * N + i];
    __syncthreads();
    const double* Am = A + (size_t)m * N * N;
    for (int r = threadIdx.x; r < N; r += blockDim.x) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int c = 0;
      for (; c + 3 < N; c += 4) {
        a0 += __ldcs(Am + (size_t)c * N + r) * sx[c];
        a1 += __ldcs(Am + (size_t)(c + 1) * N + r) * sx[c + 1];
        a2 += __ldcs(Am + (size_t)(c + 2) * N + r) * sx[c + 2];
        a3 += __ldcs(Am + (size_t)(c + 3) * N + r) * sx[c + 3];
      }
      for (; c < N; ++c) a0 += __ldcs(Am + (size_t)c * N + r) * sx[c];
      y[(size_t)m * N + r] = (a0 + a1) + (a2 + a3);
    }
  }
}

// face blocks of the preconditioner, row-major (NB x NB) per face:
//   sum over the face's tiles of face_w fphi_i hh[s][t] fphi_j at (tidx_i s, tidx_j t)
// plus the symmetry statistic (reference assembly.py:741-742, debug count)
template <int P>
__global__ void __launch_bounds__(128)
mm_precond_blk(MGeo g, const double* __restrict__ hh, double* __restrict__ blocks, int* n_unsym) {
  using D = Dims<P>;
  constexpr int NFN = D::NFN, NQF = D::NQF;
  __shared__ double red[2][128];
  const int NB = 5 * g.nt;
  const int tid = threadIdx.x;
  for (int f = blockIdx.x; f < g.F; f += gridDim.x) {
    double* B = blocks + (size_t)f * NB * NB;
    __syncthreads();
    for (int i = tid; i < NB * NB; i += 128) B[i] = 0.0;
    __syncthreads();
    for (int l = g.fptr[f]; l < g.fptr[f + 1]; ++l) {
      const int ek = g.flist[l];
      const int* td = g.tidx + (size_t)ek * NFN;
      const double ar = g.area[ek];
      const double* h = hh + (size_t)ek * NQF * 25;
      for (int ijp = tid; ijp < NFN * NFN; ijp += 128) {
        const int i = ijp / NFN, j = ijp % NFN;
        double acc[25];
#pragma unroll
        for (int st = 0; st < 25; ++st) acc[st] = 0.0;
        for (int q = 0; q < NQF; ++q) {
          const double ci = (g.fw[q] * ar) * g.fphi[q * NFN + i], pj = g.fphi[q * NFN + j];
#pragma unroll
          for (int st = 0; st < 25; ++st) acc[st] += (ci * h[q * 25 + st]) * pj;
        }
        const int ri = td[i] * 5, cj = td[j] * 5;
#pragma unroll
        for (int st = 0; st < 25; ++st) B[(size_t)(ri + st / 5) * NB + cj + st % 5] += acc[st];
      }
      __syncthreads();
    }
    double amax = 0.0, dmax = 0.0;
    for (int i = tid; i < NB * NB; i += 128) {
      const int r = i / NB, c = i % NB;
      amax = fmax(amax, fabs(B[i]));
      dmax = fmax(dmax, fabs(B[i] - B[(size_t)c * NB + r]));
    }
    red[0][tid] = amax;
    red[1][tid] = dmax;
    __syncthreads();
    for (int sft = 64; sft > 0; sft >>= 1) {
      if (tid < sft) {
        red[0][tid] = fmax(red[0][tid], red[0][tid + sft]);
        red[1][tid] = fmax(red[1][tid], red[1][tid + sft]);
      }
      __syncthreads();
    }
    if (tid == 0 && !(red[1][0] <= 1e-12 * fmax(1.0, red[0][0]))) atomicAdd(n_unsym, 1);
  }
}

}  // namespace mhdg
