// Device kernels of the macro-element HDG operator (m = 1, 3D, degree P).
//
// Data layout in HBM (float64, reference layouts so inputs are drop-in):
//   w       (E, NN, 5)      nodal working variables per macro
//   trace   (F, NFN, 5)     trace nodes per skeleton face (owner order)
//   offset  (E, NQ, 5)      stage offset at volume quadrature points
//   sinv    (E, NM, NM)     S^-1 per macro, column-major  (NM = 5 NN)
//   hw/hhat/hh (E, 4, NQF, 5, 5) face-quadrature linearization tensors
//   pinv    (F, NB, NB)     face-block inverse, column-major (NB = 5 NFN)
// Per-macro geometry (det, J^-1, normals, areas, face ids, trace
// permutations) is uploaded once; basis tables are staged in shared memory
// once per persistent CTA.
//
// Trace scatter: with m = 1 every trace node receives exactly two side
// contributions (one per skeleton side) on a zeroed output, so fp64
// atomicAdd yields 0 + a + b = the reference's np.add.at sum bit for bit
// and independent of order (IEEE addition is commutative).
#pragma once
#include "mhdg_math.cuh"
#include "mhdg_tma.cuh"

namespace mhdg {

template <int P>
struct Dims {
  static constexpr int NN = (P + 1) * (P + 2) * (P + 3) / 6;
  static constexpr int NQ = (P + 1) * (P + 1) * (P + 1);
  static constexpr int NFN = (P + 1) * (P + 2) / 2;
  static constexpr int NQF = (P + 1) * (P + 1);
  static constexpr int NM = 5 * NN;
  static constexpr int NB = 5 * NFN;
  // odd strides avoid shared-memory bank conflicts for per-q row access
  static constexpr int QS = 4 * NN + 1;                  // B table row (q)
  static constexpr int FS = (NFN % 2) ? NFN : NFN + 1;   // facet table row
  static constexpr int GS = 21;                          // volume flux row
};

struct Geo {
  int E, F;
  int form, kind;
  double gamma;
  // reference tables
  const double* B;     // (NQ, 4, NN): dphi_x, dphi_y, dphi_z, phi
  const double* qw;    // (NQ)
  const double* pf;    // (4, NQF, NFN)
  const double* fphi;  // (NQF, NFN)
  const double* fw;    // (NQF)
  const int* rows;     // (4, NFN)
  const int* nodef;    // (NN, 3): k*NFN+j of faces containing node, -1 pad
  // per macro
  const double* det;   // (E)
  const double* invj;  // (E, 9)  [k][a]
  const double* nrm;   // (E, 4, 3)
  const double* area;  // (E, 4)
  const int* fid;      // (E, 4)
  const int* tidx;     // (E, 4, NFN)
  const unsigned char* bnd;  // (E, 4)
  const int* fsides;   // (F, 2)
  int has_uinf;
  double uinf[5];
};

// status key: ((loc*4 + sub) << 40) | item ; smallest key = first error in
// the reference's loop order (volume sub, then tiles; entropy before check)
__device__ __forceinline__ void report(unsigned long long* st, int loc, int sub, long long item) {
  unsigned long long key = ((unsigned long long)(loc * 4 + sub) << 40) | (unsigned long long)item;
  atomicMin(st, key);
}

template <int P>
struct Smem {
  using D = Dims<P>;
  static constexpr int tables = D::NQ * D::QS + 4 * D::NQF * D::FS + D::NQF * D::FS + D::NQ + D::NQF;
};

// Stage reference tables into shared memory.
template <int P>
__device__ void load_tables(const Geo& g, double* sB, double* sPF, double* sFP, double* sQW,
                            double* sFW, int* sRows, int* sNF) {
  using D = Dims<P>;
  for (int i = threadIdx.x; i < D::NQ * 4 * D::NN; i += blockDim.x) {
    int q = i / (4 * D::NN), r = i % (4 * D::NN);
    sB[q * D::QS + r] = g.B[i];
  }
  for (int i = threadIdx.x; i < 4 * D::NQF * D::NFN; i += blockDim.x) {
    int kq = i / D::NFN, j = i % D::NFN;
    sPF[kq * D::FS + j] = g.pf[i];
  }
  for (int i = threadIdx.x; i < D::NQF * D::NFN; i += blockDim.x) {
    int q = i / D::NFN, j = i % D::NFN;
    sFP[q * D::FS + j] = g.fphi[i];
  }
  for (int i = threadIdx.x; i < D::NQ; i += blockDim.x) sQW[i] = g.qw[i];
  for (int i = threadIdx.x; i < D::NQF; i += blockDim.x) sFW[i] = g.fw[i];
  if (sRows)
    for (int i = threadIdx.x; i < 4 * D::NFN; i += blockDim.x) sRows[i] = g.rows[i];
  if (sNF)
    for (int i = threadIdx.x; i < 3 * D::NN; i += blockDim.x) sNF[i] = g.nodef[i];
}

// ===========================================================================
// K1: residual  (assembly.py:459-549, inviscid)
//
// Persistent CTAs, EB macros per iteration.  Phases:
//  1. pointwise: every thread evaluates one face and one volume quadrature
//     point per macro (balanced), producing the weighted two-point fluxes
//     H[k][q][s] and the reference-space flux / temporal rows G[q][kk][s]
//     (kk = 0..2: -vol_w J^-1 F, kk = 3: vol_w (alpha u + offset));
//  2. contraction, warp-specialized per macro:
//     DMMA warps: r_w^T (5 x NN) = G^T (5 x 4NQ) . B (4NQ x NN) on the FP64
//       tensor cores (mma.sync.m8n8k4.f64, SASS DMMA), K split across warps;
//     face warps: face tests of r_w (phi_face) and the side contributions to
//       r_trace (fphi), scattered with fp64 atomics (two sides per trace
//       node on a zeroed output: 0 + a + b, order independent);
//  3. r_w = volume part + face parts in tile order.
// The basis table B (NQ x 4 x NN) is read through L1 (__ldg).
// ===========================================================================
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int P>
struct ResCfg {
  using D = Dims<P>;
  static constexpr int EB = (P >= 4) ? 1 : 2;      // macros per CTA iteration
  static constexpr int NW = (P >= 4) ? 8 : 4;      // warps per CTA
  static constexpr int NT = NW * 32;
  static constexpr int WPM = NW / EB;              // warps per macro
  static constexpr int DW = WPM / 2;               // DMMA warps per macro (K split)
  static constexpr int FW = WPM - DW;              // face warps per macro
  static constexpr int NTILE = (D::NN + 7) / 8;    // DMMA N tiles over nodes
  static constexpr int GS = 21;                    // G row stride (odd)
  static constexpr int W_ = D::NN * 5, TR_ = 4 * D::NFN * 5, G_ = D::NQ * GS, H_ = 4 * D::NQF * 5,
                       FR_ = 4 * D::NFN * 5, VOL_ = DW * D::NN * 5, GEO_ = 26;
  static constexpr int per_macro = W_ + TR_ + G_ + 2 * H_ + FR_ + VOL_ + GEO_;
  static constexpr int tables = 4 * D::NQF * D::FS + D::NQF * D::FS + D::NQ + D::NQF;
  static constexpr int per_macro_int = 4 + 4 * D::NFN + 4;
  static constexpr int table_int = 4 * D::NFN + 3 * D::NN;
  static constexpr size_t bytes =
      (size_t)(tables + EB * per_macro) * 8 + (size_t)(table_int + EB * per_macro_int) * 4;
};

template <int P>
__global__ void __launch_bounds__(ResCfg<P>::NT, 512 / ResCfg<P>::NT)
k_residual(Geo g, const double* __restrict__ w, const double* __restrict__ trace,
           int has_stage, double alpha, const double* __restrict__ offset, int check,
           double* __restrict__ r_w, double* __restrict__ r_tr, unsigned long long* status) {
  using D = Dims<P>;
  using R = ResCfg<P>;
  constexpr int NT = R::NT, EB = R::EB, NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF;
  constexpr int GS = R::GS;
  extern __shared__ __align__(16) double smem[];
  double* sPF = smem;                              // 4*NQF*FS
  double* sFP = sPF + 4 * NQF * D::FS;             // NQF*FS
  double* sQW = sFP + NQF * D::FS;                 // NQ
  double* sFW = sQW + NQ;                          // NQF
  double* mb = sFW + NQF;                          // EB * per_macro
  int* sRows = (int*)(mb + EB * R::per_macro);     // 4*NFN
  int* sNF = sRows + 4 * NFN;                      // 3*NN
  int* ib = sNF + 3 * NN;                          // EB * per_macro_int
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 4 * NQF * NFN; i += NT) sPF[(i / NFN) * D::FS + i % NFN] = g.pf[i];
  for (int i = tid; i < NQF * NFN; i += NT) sFP[(i / NFN) * D::FS + i % NFN] = g.fphi[i];
  for (int i = tid; i < NQ; i += NT) sQW[i] = g.qw[i];
  for (int i = tid; i < NQF; i += NT) sFW[i] = g.fw[i];
  for (int i = tid; i < 4 * NFN; i += NT) sRows[i] = g.rows[i];
  for (int i = tid; i < 3 * NN; i += NT) sNF[i] = g.nodef[i];
  const double gam = g.gamma;
  const double* __restrict__ Bt = g.B;

  auto W = [&](int m) { return mb + m * R::per_macro; };
  auto TR = [&](int m) { return W(m) + R::W_; };
  auto G = [&](int m) { return TR(m) + R::TR_; };
  auto H = [&](int m) { return G(m) + R::G_; };
  auto HG = [&](int m) { return H(m) + R::H_; };
  auto FR = [&](int m) { return HG(m) + R::H_; };
  auto VOL = [&](int m) { return FR(m) + R::FR_; };
  auto GEO = [&](int m) { return VOL(m) + R::VOL_; };
  auto FID = [&](int m) { return ib + m * R::per_macro_int; };
  auto TID = [&](int m) { return FID(m) + 4; };
  auto BND = [&](int m) { return TID(m) + 4 * NFN; };

  for (int e0 = blockIdx.x * EB; e0 < g.E; e0 += gridDim.x * EB) {
    const int nm = min(EB, g.E - e0);
    __syncthreads();
    for (int i = tid; i < nm * NN * 5; i += NT) W(i / (NN * 5))[i % (NN * 5)] = w[(size_t)e0 * NN * 5 + i];
    for (int i = tid; i < nm * 4; i += NT) {
      const int m = i / 4, k = i % 4, e = e0 + m;
      FID(m)[k] = g.fid[e * 4 + k];
      BND(m)[k] = g.bnd ? g.bnd[e * 4 + k] : 0;
    }
    for (int i = tid; i < nm * 4 * NFN; i += NT) {
      const int m = i / (4 * NFN);
      TID(m)[i % (4 * NFN)] = g.tidx[(size_t)e0 * 4 * NFN + i];
    }
    for (int i = tid; i < nm * 26; i += NT) {
      const int m = i / 26, c = i % 26, e = e0 + m;
      double v;
      if (c == 0) v = g.det[e];
      else if (c < 10) v = g.invj[(size_t)e * 9 + c - 1];
      else if (c < 22) v = g.nrm[(size_t)e * 12 + c - 10];
      else v = g.area[(size_t)e * 4 + c - 22];
      GEO(m)[c] = v;
    }
    __syncthreads();
    for (int i = tid; i < nm * 4 * NFN * 5; i += NT) {
      const int m = i / (4 * NFN * 5), r = i % (4 * NFN * 5);
      const int k = r / (NFN * 5), j = (r / 5) % NFN, s = r % 5;
      TR(m)[r] = trace[((size_t)FID(m)[k] * NFN + TID(m)[k * NFN + j]) * 5 + s];
    }
    __syncthreads();

    // ---- 1a. face quadrature points: two-point flux, weighted
    for (int it = tid; it < nm * 4 * NQF; it += NT) {
      const int m = it / (4 * NQF), kq = it % (4 * NQF), k = kq / NQF, q = kq % NQF, e = e0 + m;
      const double* pf = sPF + kq * D::FS;
      const double* fp = sFP + q * D::FS;
      const double* sw = W(m);
      const double* st = TR(m) + k * NFN * 5;
      double wq[5] = {0, 0, 0, 0, 0}, whq[5] = {0, 0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < NFN; ++j) {
        const double a = pf[j], b = fp[j];
        const int row = sRows[k * NFN + j];
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          wq[s] += a * sw[row * 5 + s];
          whq[s] += b * st[j * 5 + s];
        }
      }
      double u[5], uh[5];
      if (!to_conservative(wq, g.form, gam, u)) report(status, 1 + k, 0, e);
      if (!to_conservative(whq, g.form, gam, uh)) report(status, 1 + k, 1, e);
      if (check && !admissible(u, gam)) report(status, 1 + k, 2, e);
      if (check && !admissible(uh, gam)) report(status, 1 + k, 3, e);
      const double* geo = GEO(m);
      const double n[3] = {geo[10 + k * 3], geo[11 + k * 3], geo[12 + k * 3]};
      double fh[5];
      numerical_flux(g.kind, u, uh, n, gam, fh);
      const double fwq = sFW[q] * geo[22 + k];
      double* h = H(m) + kq * 5;
#pragma unroll
      for (int s = 0; s < 5; ++s) h[s] = fwq * fh[s];
      if (BND(m)[k] && g.has_uinf) {
        const double mn[3] = {-n[0], -n[1], -n[2]};
        double gh[5];
        numerical_flux(g.kind, g.uinf, uh, mn, gam, gh);
#pragma unroll
        for (int s = 0; s < 5; ++s) HG(m)[kq * 5 + s] = fwq * gh[s];
      }
    }
    // ---- 1b. volume quadrature points: reference-space flux + temporal term
    for (int it = tid; it < nm * NQ; it += NT) {
      const int m = it / NQ, q = it % NQ, e = e0 + m;
      const double* ph = Bt + ((size_t)q * 4 + 3) * NN;
      const double* sw = W(m);
      double wq[5] = {0, 0, 0, 0, 0};
#pragma unroll 4
      for (int i = 0; i < NN; ++i) {
        const double a = __ldg(ph + i);
#pragma unroll
        for (int s = 0; s < 5; ++s) wq[s] += a * sw[i * 5 + s];
      }
      double u[5];
      if (!to_conservative(wq, g.form, gam, u)) report(status, 0, 0, e);
      if (check && !admissible(u, gam)) report(status, 0, 2, e);
      double F[5][3];
      flux(u, gam, F);
      const double* geo = GEO(m);
      const double vw = sQW[q] * geo[0];
      double* gr = G(m) + q * GS;
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) {
        const double j0 = geo[1 + kk * 3], j1 = geo[2 + kk * 3], j2 = geo[3 + kk * 3];
#pragma unroll
        for (int s = 0; s < 5; ++s) gr[kk * 5 + s] = -(vw * ((j0 * F[s][0] + j1 * F[s][1]) + j2 * F[s][2]));
      }
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        double tmp = 0.0;
        if (has_stage) {
          tmp = alpha * u[s];
          if (offset) tmp = tmp + offset[((size_t)e * NQ + q) * 5 + s];
          tmp = vw * tmp;
        }
        gr[15 + s] = tmp;
      }
    }
    __syncthreads();

    // ---- 2. contraction, warp-specialized per macro
    {
      const int m = warp / R::WPM, role = warp % R::WPM;
      if (m < nm) {
        if (role < R::DW) {
          // DMMA: C[s][i] += sum_k G^T[s][k] B[k][i], k = (q, kk)
          const int q0 = role * NQ / R::DW, q1 = (role + 1) * NQ / R::DW;
          const int s_a = lane >> 2, kk = lane & 3;
          double c[R::NTILE][2];
#pragma unroll
          for (int t = 0; t < R::NTILE; ++t) c[t][0] = c[t][1] = 0.0;
          const double* gm = G(m);
          for (int q = q0; q < q1; ++q) {
            const double a = s_a < 5 ? gm[q * GS + kk * 5 + s_a] : 0.0;
            const double* brow = Bt + ((size_t)q * 4 + kk) * NN;
#pragma unroll
            for (int t = 0; t < R::NTILE; ++t) {
              const int i = t * 8 + (lane >> 2);
              const double b = i < NN ? __ldg(brow + i) : 0.0;
              dmma_8x8x4(c[t], a, b);
            }
          }
          double* vol = VOL(m) + role * NN * 5;
          const int s_c = lane >> 2;
          if (s_c < 5) {
#pragma unroll
            for (int t = 0; t < R::NTILE; ++t)
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const int i = t * 8 + (lane & 3) * 2 + h2;
                if (i < NN) vol[i * 5 + s_c] = c[t][h2];
              }
          }
        } else {
          const int fr = role - R::DW, fl = fr * 32 + lane, fstride = R::FW * 32;
          const double* hm = H(m);
          const int* fid = FID(m);
          const int* tdx = TID(m);
          const bool bnd_any = g.has_uinf && (BND(m)[0] | BND(m)[1] | BND(m)[2] | BND(m)[3]);
          for (int o = fl; o < 4 * NFN * 5; o += fstride) {
            const int k = o / (NFN * 5), j = (o / 5) % NFN, s = o % 5;
            double a = 0.0, b = 0.0;
#pragma unroll 4
            for (int q = 0; q < NQF; ++q) {
              const double hv = hm[(k * NQF + q) * 5 + s];
              a += sPF[(k * NQF + q) * D::FS + j] * hv;
              b += sFP[q * D::FS + j] * hv;
            }
            FR(m)[o] = a;
            if (bnd_any && BND(m)[k]) {
              double gsum = 0.0;
              for (int q = 0; q < NQF; ++q) gsum += sFP[q * D::FS + j] * HG(m)[(k * NQF + q) * 5 + s];
              b += gsum;
            }
            atomicAdd(&r_tr[((size_t)fid[k] * NFN + tdx[k * NFN + j]) * 5 + s], b);
          }
        }
      }
    }
    __syncthreads();
    // ---- 3. r_w = volume part + face parts (tile order)
    for (int o = tid; o < nm * NN * 5; o += NT) {
      const int m = o / (NN * 5), is = o % (NN * 5), i = is / 5, s = is % 5;
      double r = VOL(m)[is];
#pragma unroll
      for (int d2 = 1; d2 < R::DW; ++d2) r += VOL(m)[d2 * NN * 5 + is];
#pragma unroll
      for (int c2 = 0; c2 < 3; ++c2) {
        const int kj = sNF[i * 3 + c2];
        if (kj < 0) break;
        r += FR(m)[kj * 5 + s];
      }
      r_w[(size_t)e0 * NN * 5 + o] = r;
    }
  }
}

// ===========================================================================
// In-place Gauss-Jordan inverse with partial (row) pivoting, n x n row-major
// in `A` (shared or global), whole block cooperating.  Pivot choice: first
// row of maximal |a_ik| (LAPACK idamax semantics).  Returns false (uniformly
// across the block) if a pivot is zero or non-finite.
// ===========================================================================
__device__ bool gj_inverse(double* A, int n, int lda, int* perm, double* col, int* sflag) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) *sflag = 0;
  for (int k = 0; k < n; ++k) {
    __syncthreads();
    if (tid < 32) {
      double best = -1.0;
      int bi = n;
      for (int r = k + tid; r < n; r += 32) {
        double v = fabs(A[r * lda + k]);
        if (v > best || (v != v && best >= 0)) { best = v; bi = r; }
      }
      for (int off = 16; off > 0; off >>= 1) {
        double ob = __shfl_down_sync(0xffffffffu, best, off);
        int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) {
        perm[k] = bi;
        double pv = bi < n ? A[bi * lda + k] : 0.0;
        if (!(fabs(pv) > 0.0) || !isfinite(pv)) *sflag = 1;
      }
    }
    __syncthreads();
    const int p = perm[k];
    if (p != k)
      for (int j = tid; j < n; j += nt) {
        double t = A[k * lda + j];
        A[k * lda + j] = A[p * lda + j];
        A[p * lda + j] = t;
      }
    __syncthreads();
    for (int r = tid; r < n; r += nt) col[r] = A[r * lda + k];
    __syncthreads();
    const double pinv = 1.0 / col[k];
    for (int j = tid; j < n; j += nt) A[k * lda + j] = (j == k ? 1.0 : A[k * lda + j]) * pinv;
    __syncthreads();
    for (int idx = tid; idx < n * n; idx += nt) {
      const int r = idx / n, j = idx % n;
      if (r == k) continue;
      const double base = (j == k) ? 0.0 : A[r * lda + j];
      A[r * lda + j] = base - A[k * lda + j] * col[r];
    }
  }
  __syncthreads();
  // undo the row interchanges as column interchanges, in reverse order
  for (int r = tid; r < n; r += nt)
    for (int k = n - 1; k >= 0; --k) {
      const int p = perm[k];
      if (p != k) {
        double t = A[r * lda + k];
        A[r * lda + k] = A[r * lda + p];
        A[r * lda + p] = t;
      }
    }
  __syncthreads();
  return *sflag == 0;
}

// ===========================================================================
// K2: linearize + assemble S + S^-1   (assembly.py:772-976)
// ===========================================================================
template <int P>
struct LinSmem {
  using D = Dims<P>;
  static constexpr int QC = 8;                                // q chunk
  static constexpr bool S_IN_SMEM = (D::NM * D::NM * 8) <= 100 * 1024;
  static constexpr int doubles =
      Smem<P>::tables + D::NN * 5 + 4 * D::NFN * 5 + QC * 100 + D::NQF * 25 + D::NM + 32 +
      (S_IN_SMEM ? D::NM * D::NM : 0);
  static constexpr int ints = 4 * D::NFN + 4 + 4 * D::NFN + 4 + D::NM + 4;
  static constexpr size_t bytes = doubles * 8 + ints * 4;
};

template <int P, int NT>
__global__ void __launch_bounds__(NT)
k_linearize(Geo g, const double* __restrict__ w, const double* __restrict__ trace, double weight,
            double ptc, double* __restrict__ sinv, double* __restrict__ hw_out,
            double* __restrict__ hhat_out, double* __restrict__ hh_out, double* __restrict__ scratch,
            unsigned long long* status) {
  using D = Dims<P>;
  using L = LinSmem<P>;
  constexpr int QC = L::QC;
  constexpr int NM = D::NM;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sPF = sB + D::NQ * D::QS;
  double* sFP = sPF + 4 * D::NQF * D::FS;
  double* sQW = sFP + D::NQF * D::FS;
  double* sFW = sQW + D::NQ;
  double* sW = sFW + D::NQF;
  double* sTR = sW + D::NN * 5;
  double* sC = sTR + 4 * D::NFN * 5;          // QC*100  [qq][kk][s][t]
  double* sHW = sC + QC * 100;                 // NQF*25
  double* sCol = sHW + D::NQF * 25;            // NM
  double* sGeo = sCol + NM;                    // 32
  double* S = L::S_IN_SMEM ? (sGeo + 32) : (scratch + (size_t)blockIdx.x * NM * NM);
  int* ibase = (int*)(sGeo + 32 + (L::S_IN_SMEM ? NM * NM : 0));
  int* sRows = ibase;
  int* sFid = sRows + 4 * D::NFN;
  int* sTid = sFid + 4;
  int* sBnd = sTid + 4 * D::NFN;
  int* sPerm = sBnd + 4;
  int* sFlag = sPerm + NM;
  load_tables<P>(g, sB, sPF, sFP, sQW, sFW, sRows, nullptr);
  const double gam = g.gamma;
  const int tid = threadIdx.x;

  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < D::NN * 5; i += NT) sW[i] = w[(size_t)e * D::NN * 5 + i];
    if (tid < 4) {
      sFid[tid] = g.fid[e * 4 + tid];
      sBnd[tid] = g.bnd ? g.bnd[e * 4 + tid] : 0;
    }
    for (int i = tid; i < 4 * D::NFN; i += NT) sTid[i] = g.tidx[(size_t)e * 4 * D::NFN + i];
    if (tid == 0) sGeo[0] = g.det[e];
    if (tid >= 1 && tid < 10) sGeo[tid] = g.invj[(size_t)e * 9 + tid - 1];
    if (tid >= 10 && tid < 22) sGeo[tid] = g.nrm[(size_t)e * 12 + tid - 10];
    if (tid >= 22 && tid < 26) sGeo[tid] = g.area[(size_t)e * 4 + tid - 22];
    for (int i = tid; i < NM * NM; i += NT) S[i] = 0.0;
    __syncthreads();
    for (int i = tid; i < 4 * D::NFN * 5; i += NT) {
      int k = i / (D::NFN * 5), j = (i / 5) % D::NFN, s = i % 5;
      sTR[i] = trace[((size_t)sFid[k] * D::NFN + sTid[k * D::NFN + j]) * 5 + s];
    }

    // ---- volume blocks, in chunks of QC quadrature points
    for (int q0 = 0; q0 < D::NQ; q0 += QC) {
      __syncthreads();
      for (int it = tid; it < QC * 5; it += NT) {
        const int qq = it / 5, t = it % 5, q = q0 + qq;
        double* C = sC + qq * 100;
        if (q >= D::NQ) {
          for (int r = 0; r < 4; ++r)
            for (int s = 0; s < 5; ++s) C[r * 25 + s * 5 + t] = 0.0;
          continue;
        }
        const double* Bq = sB + q * D::QS + 3 * D::NN;
        double wq[5] = {0, 0, 0, 0, 0};
        for (int i = 0; i < D::NN; ++i) {
          double ph = Bq[i];
#pragma unroll
          for (int s = 0; s < 5; ++s) wq[s] += ph * sW[i * 5 + s];
        }
        Dual wd[5], ud[5];
#pragma unroll
        for (int s = 0; s < 5; ++s) wd[s] = mk(wq[s], s == t ? 1.0 : 0.0);
        to_conservative(wd, g.form, gam, ud);
        Dual F[5][3];
        flux(ud, gam, F);
        const double vw = sQW[q] * sGeo[0];
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const double j0 = sGeo[1 + kk * 3], j1 = sGeo[2 + kk * 3], j2 = sGeo[3 + kk * 3];
#pragma unroll
          for (int s = 0; s < 5; ++s)
            C[kk * 25 + s * 5 + t] = -(vw * ((j0 * F[s][0].d + j1 * F[s][1].d) + j2 * F[s][2].d));
        }
#pragma unroll
        for (int s = 0; s < 5; ++s) C[75 + s * 5 + t] = weight * (vw * ud[s].d);
      }
      __syncthreads();
      const int qn = (D::NQ - q0) < QC ? (D::NQ - q0) : QC;
      for (int o = tid; o < NM * NM; o += NT) {
        const int r = o / NM, c = o % NM;
        const int i = r / 5, s = r % 5, j = c / 5, t = c % 5;
        double acc = 0.0;
        for (int qq = 0; qq < qn; ++qq) {
          const double* Bq = sB + (q0 + qq) * D::QS;
          const double* C = sC + qq * 100 + s * 5 + t;
          const double dd = ((Bq[i] * C[0] + Bq[D::NN + i] * C[25]) + Bq[2 * D::NN + i] * C[50]) +
                            Bq[3 * D::NN + i] * C[75];
          acc += dd * Bq[3 * D::NN + j];
        }
        S[o] += acc;
      }
    }

    // ---- face tiles: hw, hhat, hh tensors and the S face blocks
    for (int k = 0; k < 4; ++k) {
      __syncthreads();
      const double n[3] = {sGeo[10 + k * 3], sGeo[11 + k * 3], sGeo[12 + k * 3]};
      for (int it = tid; it < D::NQF * 10; it += NT) {
        const int q = it / 10, t = (it % 10) % 5, which = (it % 10) / 5;
        const double* pf = sPF + (k * D::NQF + q) * D::FS;
        const double* fp = sFP + q * D::FS;
        double wq[5] = {0, 0, 0, 0, 0}, whq[5] = {0, 0, 0, 0, 0};
        for (int j = 0; j < D::NFN; ++j) {
          const double a = pf[j], b = fp[j];
          const int row = sRows[k * D::NFN + j];
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            wq[s] += a * sW[row * 5 + s];
            whq[s] += b * sTR[(k * D::NFN + j) * 5 + s];
          }
        }
        Dual wd[5], whd[5], ud[5], uhd[5], fd[5];
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          wd[s] = mk(wq[s], (which == 0 && s == t) ? 1.0 : 0.0);
          whd[s] = mk(whq[s], (which == 1 && s == t) ? 1.0 : 0.0);
        }
        to_conservative(wd, g.form, gam, ud);
        to_conservative(whd, g.form, gam, uhd);
        numerical_flux(g.kind, ud, uhd, n, gam, fd);
        const size_t base = (((size_t)e * 4 + k) * D::NQF + q) * 25;
        if (which == 0) {
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            hw_out[base + s * 5 + t] = fd[s].d;
            sHW[q * 25 + s * 5 + t] = fd[s].d;
          }
        } else {
          double hh[5];
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            hhat_out[base + s * 5 + t] = fd[s].d;
            hh[s] = fd[s].d;
          }
          if (sBnd[k] && g.has_uinf) {
            Dual ui[5], gd[5];
#pragma unroll
            for (int s = 0; s < 5; ++s) ui[s] = mk(g.uinf[s], 0.0);
            const double mn[3] = {-n[0], -n[1], -n[2]};
            numerical_flux(g.kind, ui, uhd, mn, gam, gd);
#pragma unroll
            for (int s = 0; s < 5; ++s) hh[s] = hh[s] + gd[s].d;
          }
          if (ptc != 0.0) {
#pragma unroll
            for (int s = 0; s < 5; ++s) hh[s] = hh[s] + (-ptc * uhd[s].d);
          }
#pragma unroll
          for (int s = 0; s < 5; ++s) hh_out[base + s * 5 + t] = hh[s];
        }
      }
      __syncthreads();
      const double ar = sGeo[22 + k];
      for (int o = tid; o < D::NFN * D::NFN * 25; o += NT) {
        const int ij = o / 25, st = o % 25;
        const int i = ij / D::NFN, j = ij % D::NFN, s = st / 5, t = st % 5;
        double acc = 0.0;
        for (int q = 0; q < D::NQF; ++q) {
          const double* pf = sPF + (k * D::NQF + q) * D::FS;
          acc += (((sFW[q] * ar) * pf[i]) * sHW[q * 25 + st]) * pf[j];
        }
        const int r = sRows[k * D::NFN + i] * 5 + s, c = sRows[k * D::NFN + j] * 5 + t;
        S[r * NM + c] += acc;
      }
    }
    __syncthreads();

    // ---- S^-1 (Gauss-Jordan) and column-major store
    bool ok = gj_inverse(S, NM, NM, sPerm, sCol, sFlag);
    int bad = 0;
    for (int o = tid; o < NM * NM; o += NT) bad |= !isfinite(S[o]);
    bad = __syncthreads_or(bad);
    if ((!ok || bad) && tid == 0) report(status, 0, 0, e);
    double* out = sinv + (size_t)e * NM * NM;
    for (int o = tid; o < NM * NM; o += NT) {
      const int c = o / NM, r = o % NM;
      out[o] = S[r * NM + c];
    }
  }
}

// ===========================================================================
// K4 (factor): face-block preconditioner  (assembly.py:994-1026, 736-752)
// ===========================================================================
template <int P, int NT>
__global__ void __launch_bounds__(NT)
k_precond_factor(Geo g, int n_faces, const double* __restrict__ hh, const double* __restrict__ hh_rem,
                 const int* __restrict__ tidx_rem, const double* __restrict__ area_rem,
                 double* __restrict__ pinv, unsigned long long* status, int* n_unsym) {
  using D = Dims<P>;
  constexpr int NB = D::NB;
  extern __shared__ double smem[];
  double* A = smem;                      // NB*NB
  double* sHH = A + NB * NB;             // NQF*25
  double* sFP = sHH + D::NQF * 25;       // NQF*NFN
  double* sCol = sFP + D::NQF * D::NFN;  // NB
  double* sFw = sCol + NB;               // NQF
  int* sT = (int*)(sFw + D::NQF);        // NFN
  int* sPerm = sT + D::NFN;              // NB
  int* sFlag = sPerm + NB;               // 2
  const int tid = threadIdx.x;
  for (int i = tid; i < D::NQF * D::NFN; i += NT) sFP[i] = g.fphi[i];
  for (int f = blockIdx.x; f < n_faces; f += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < NB * NB; i += NT) A[i] = 0.0;
    for (int side = 0; side < 2; ++side) {
      const int st = g.fsides[f * 2 + side];
      if (st == -1) continue;
      __syncthreads();
      if (st >= 0) {
        const int e = st / 4, k = st % 4;
        for (int i = tid; i < D::NQF * 25; i += NT) sHH[i] = hh[((size_t)st * D::NQF) * 25 + i];
        for (int i = tid; i < D::NFN; i += NT) sT[i] = g.tidx[((size_t)e * 4 + k) * D::NFN + i];
        for (int i = tid; i < D::NQF; i += NT) sFw[i] = g.fw[i] * g.area[(size_t)e * 4 + k];
      } else {  // remote side of a halo face (partitioned runs)
        const int r = -2 - st;
        for (int i = tid; i < D::NQF * 25; i += NT) sHH[i] = hh_rem[(size_t)r * D::NQF * 25 + i];
        for (int i = tid; i < D::NFN; i += NT) sT[i] = tidx_rem[(size_t)r * D::NFN + i];
        for (int i = tid; i < D::NQF; i += NT) sFw[i] = g.fw[i] * area_rem[r];
      }
      __syncthreads();
      for (int o = tid; o < D::NFN * D::NFN * 25; o += NT) {
        const int ij = o / 25, stt = o % 25;
        const int i = ij / D::NFN, j = ij % D::NFN, s = stt / 5, t = stt % 5;
        double acc = 0.0;
        for (int q = 0; q < D::NQF; ++q)
          acc += ((sFw[q] * sFP[q * D::NFN + i]) * sHH[q * 25 + stt]) * sFP[q * D::NFN + j];
        A[(sT[i] * 5 + s) * NB + sT[j] * 5 + t] += acc;
      }
    }
    __syncthreads();
    // symmetry statistic (reference logs the count of non-SPD/non-symmetric blocks)
    if (tid < 32) {
      double amax = 0.0, dmax = 0.0;
      for (int idx = tid; idx < NB * NB; idx += 32) {
        const int r = idx / NB, c = idx % NB;
        amax = fmax(amax, fabs(A[idx]));
        dmax = fmax(dmax, fabs(A[idx] - A[c * NB + r]));
      }
      for (int off = 16; off > 0; off >>= 1) {
        amax = fmax(amax, __shfl_down_sync(0xffffffffu, amax, off));
        dmax = fmax(dmax, __shfl_down_sync(0xffffffffu, dmax, off));
      }
      if (tid == 0 && !(dmax <= 1e-12 * fmax(1.0, amax))) atomicAdd(n_unsym, 1);
    }
    bool ok = gj_inverse(A, NB, NB, sPerm, sCol, sFlag);
    int bad = 0;
    for (int o = tid; o < NB * NB; o += NT) bad |= !isfinite(A[o]);
    bad = __syncthreads_or(bad);
    if ((!ok || bad) && tid == 0) report(status, 0, 0, f);
    double* out = pinv + (size_t)f * NB * NB;
    for (int o = tid; o < NB * NB; o += NT) {
      const int c = o / NB, r = o % NB;
      out[o] = A[r * NB + c];
    }
  }
}

// ===========================================================================
// K3 / K6 as three streaming kernels (the operator is HBM-bound; splitting
// costs ~3% extra traffic -- g and z round trips -- and lets every kernel
// run many independent CTAs per SM):
//   k_face_in  : g = -(A_vh x) [matvec] or -r_w - A_vh x [recover]
//                (hhat at face quadrature points, tested with phi_face)
//   k_local_solve: z = S^-1 g, batched column-major GEMV (rhs: g = -r_w)
//   k_face_out : y += A_hh x [matvec] + A_hv z, scattered to the trace with
//                fp64 atomics (two sides per node on a zeroed output)
// ===========================================================================
// z_e = S_e^-1 g_e (column-major S^-1); neg: g = -gin (condensed rhs)
template <int NM, int NT>
__global__ void __launch_bounds__(NT)
k_local_solve(int E, const double* __restrict__ sinv, const double* __restrict__ gin, int neg,
              double* __restrict__ z) {
  __shared__ double sg[NM];
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < NM; i += NT) sg[i] = neg ? -gin[(size_t)e * NM + i] : gin[(size_t)e * NM + i];
    __syncthreads();
    const double* A = sinv + (size_t)e * NM * NM;
    for (int r = threadIdx.x; r < NM; r += NT) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int c = 0;
      for (; c + 3 < NM; c += 4) {
        a0 += __ldcs(A + (size_t)(c + 0) * NM + r) * sg[c + 0];
        a1 += __ldcs(A + (size_t)(c + 1) * NM + r) * sg[c + 1];
        a2 += __ldcs(A + (size_t)(c + 2) * NM + r) * sg[c + 2];
        a3 += __ldcs(A + (size_t)(c + 3) * NM + r) * sg[c + 3];
      }
      for (; c < NM; ++c) a0 += __ldcs(A + (size_t)c * NM + r) * sg[c];
      z[(size_t)e * NM + r] = (a0 + a1) + (a2 + a3);
    }
  }
}

// Software-pipelined face kernels: while macro e is computed from shared
// memory, every thread already holds in registers its share of macro
// e+G's face tensors and trace values (G = grid size), and the metadata
// (face ids, trace permutations, areas) of macro e+2G -- so none of the
// three dependent global round trips sits on the critical path.
template <int P, int NT>
struct FacePipe {
  using D = Dims<P>;
  static constexpr int NI = 4 * D::NQF;
  static constexpr int NTEN = NI * 25;
  static constexpr int NX = 4 * D::NFN * 5;
  static constexpr int TPT = (NTEN + NT - 1) / NT;   // tensor doubles / thread
  static constexpr int XPT = (NX + NT - 1) / NT;
  static constexpr int ZPT = (D::NM + NT - 1) / NT;
  static constexpr int META = 4 + 4 * D::NFN;        // ints: fid, tidx
  static constexpr int MPT = (META + 4 + NT - 1) / NT;
  static constexpr int doubles = 4 * D::NQF * D::FS + D::NQF * D::FS + D::NQF + NX + 2 * NTEN + D::NM +
                                 4 * NI * 5 + 3 * 4;
  static constexpr int ints = 4 * D::NFN + 3 * D::NN + 3 * META;
  static constexpr size_t bytes = (size_t)doubles * 8 + ints * 4;
};

template <int P, int NT, int MODE>   // MODE 0: face_in (A_vh x), 1: face_out (A_hh x + A_hv z)
__global__ void __launch_bounds__(NT)
k_face_pipe(Geo g, int mode, const double* __restrict__ tenA, const double* __restrict__ tenB,
            const double* __restrict__ x, const double* __restrict__ zin, const double* __restrict__ r_w,
            double* __restrict__ out) {
  using D = Dims<P>;
  using FP = FacePipe<P, NT>;
  constexpr int NM = D::NM, NFN = D::NFN, NQF = D::NQF, NN = D::NN, NI = FP::NI, NTEN = FP::NTEN,
                NX = FP::NX, META = FP::META;
  // face_in : tenA = hhat; needs x.              out = g (E, NM)
  // face_out: tenA = hw (z side), tenB = hh (x side, matvec only); out = y
  const bool use_x = (MODE == 0) || mode == 0;
  const bool use_b = (MODE == 1) && mode == 0;
  extern __shared__ __align__(16) double smem[];
  double* sPF = smem;
  double* sFP = sPF + 4 * NQF * D::FS;
  double* sFW = sFP + NQF * D::FS;
  double* sX = sFW + NQF;          // NX
  double* sTA = sX + NX;           // NTEN
  double* sTB = sTA + NTEN;        // NTEN
  double* sZ = sTB + NTEN;         // NM
  double* sQ1 = sZ + NM;           // NI*5
  double* sQ2 = sQ1 + NI * 5;      // NI*5
  double* sQ3 = sQ2 + NI * 5;      // NI*5
  double* sQ4 = sQ3 + NI * 5;      // NI*5
  double* sAr = sQ4 + NI * 5;      // 3 x 4
  int* sRows = (int*)(sAr + 12);
  int* sNF = sRows + 4 * NFN;
  int* sMeta = sNF + 3 * NN;       // 3 x META
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * NQF * NFN; i += NT) sPF[(i / NFN) * D::FS + i % NFN] = g.pf[i];
  for (int i = tid; i < NQF * NFN; i += NT) sFP[(i / NFN) * D::FS + i % NFN] = g.fphi[i];
  for (int i = tid; i < NQF; i += NT) sFW[i] = g.fw[i];
  for (int i = tid; i < 4 * NFN; i += NT) sRows[i] = g.rows[i];
  for (int i = tid; i < 3 * NN; i += NT) sNF[i] = g.nodef[i];
  const int G = gridDim.x;
  // metadata element i of macro e: i < 4 fid, < META tidx, else area (double)
  auto meta_load = [&](int e, int i, int& iv, double& dv) {
    if (i < 4) iv = g.fid[e * 4 + i];
    else if (i < META) iv = g.tidx[(size_t)e * 4 * NFN + i - 4];
    else if (i < META + 4) dv = g.area[(size_t)e * 4 + i - META];
  };
  auto meta_store = [&](int slot, int i, int iv, double dv) {
    if (i < META) sMeta[slot * META + i] = iv;
    else if (i < META + 4) sAr[slot * 4 + i - META] = dv;
  };
  // prologue: metadata of e0 and e0+G in slots 0, 1
  const int e0 = blockIdx.x;
  for (int c = 0; c < 2; ++c) {
    const int e = e0 + c * G;
    if (e < g.E)
      for (int i = tid; i < META + 4; i += NT) {
        int iv = 0;
        double dv = 0.0;
        meta_load(e, i, iv, dv);
        meta_store(c, i, iv, dv);
      }
  }
  __syncthreads();
  double rA[FP::TPT], rB[FP::TPT], rX[FP::XPT], rZ[FP::ZPT], rMd[FP::MPT];
  int rMi[FP::MPT];
  auto prefetch = [&](int e, int slot) {  // tensors / x / z of macro e (meta in slot)
    const int* mt = sMeta + slot * META;
#pragma unroll
    for (int c = 0; c < FP::TPT; ++c) {
      const int i = tid + c * NT;
      if (i < NTEN) {
        rA[c] = __ldcs(tenA + (size_t)e * NTEN + i);
        if (use_b) rB[c] = __ldcs(tenB + (size_t)e * NTEN + i);
      }
    }
    if (use_x) {
#pragma unroll
      for (int c = 0; c < FP::XPT; ++c) {
        const int i = tid + c * NT;
        if (i < NX) {
          const int k = i / (NFN * 5), j = (i / 5) % NFN, s = i % 5;
          rX[c] = x[((size_t)mt[k] * NFN + mt[4 + k * NFN + j]) * 5 + s];
        }
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int c = 0; c < FP::ZPT; ++c) {
        const int i = tid + c * NT;
        if (i < NM) rZ[c] = zin[(size_t)e * NM + i];
      }
    }
  };
  if (e0 < g.E) prefetch(e0, 0);
  int slot = 0;
  for (int e = e0; e < g.E; e += G, slot = (slot + 1) % 3) {
    const int e1 = e + G, e2 = e + 2 * G;
    const int s1 = (slot + 1) % 3, s2 = (slot + 2) % 3;
    __syncthreads();   // previous macro's compute finished with the buffers
#pragma unroll
    for (int c = 0; c < FP::TPT; ++c) {
      const int i = tid + c * NT;
      if (i < NTEN) {
        sTA[i] = rA[c];
        if (use_b) sTB[i] = rB[c];
      }
    }
    if (use_x) {
#pragma unroll
      for (int c = 0; c < FP::XPT; ++c) {
        const int i = tid + c * NT;
        if (i < NX) sX[i] = rX[c];
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int c = 0; c < FP::ZPT; ++c) {
        const int i = tid + c * NT;
        if (i < NM) sZ[i] = rZ[c];
      }
    }
    __syncthreads();
    // requests for the next macros (consumed one iteration later)
    if (e1 < g.E) prefetch(e1, s1);
    if (e2 < g.E) {
#pragma unroll
      for (int c = 0; c < FP::MPT; ++c) {
        const int i = tid + c * NT;
        rMi[c] = 0;
        rMd[c] = 0.0;
        if (i < META + 4) meta_load(e2, i, rMi[c], rMd[c]);
      }
    }
    const int* mt = sMeta + slot * META;
    const double* ar = sAr + slot * 4;
    // ---- compute macro e from shared memory
    for (int it = tid; it < NI * 5; it += NT) {
      const int kq = it / 5, t = it % 5, k = kq / NQF, q = kq % NQF;
      if (use_x) {
        const double* fp = sFP + q * D::FS;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NFN; ++j) acc += fp[j] * sX[(k * NFN + j) * 5 + t];
        sQ1[it] = acc;
      }
      if (MODE == 1) {
        const double* pf = sPF + kq * D::FS;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < NFN; ++j) acc += pf[j] * sZ[sRows[k * NFN + j] * 5 + t];
        sQ2[it] = acc;
      }
    }
    __syncthreads();
    for (int it = tid; it < NI * 5; it += NT) {
      const int kq = it / 5, s = it % 5, k = kq / NQF, q = kq % NQF;
      const double fwq = sFW[q] * ar[k];
      const double* xq = sQ1 + kq * 5;
      const double* ta = sTA + kq * 25 + s * 5;
      if (MODE == 0) {
        double a = 0.0;
#pragma unroll
        for (int t = 0; t < 5; ++t) a += ta[t] * xq[t];
        sQ3[it] = fwq * a;
      } else {
        const double* zq = sQ2 + kq * 5;
        const double* tb = sTB + kq * 25 + s * 5;
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          a += ta[t] * zq[t];
          if (use_b) b += tb[t] * xq[t];
        }
        sQ3[it] = fwq * a;
        if (use_b) sQ4[it] = fwq * b;
      }
    }
    __syncthreads();
    if (MODE == 0) {
      for (int o = tid; o < NX; o += NT) {
        const int k = o / (NFN * 5), j = (o / 5) % NFN, s = o % 5;
        double acc = 0.0;
#pragma unroll 4
        for (int q = 0; q < NQF; ++q) acc += sPF[(k * NQF + q) * D::FS + j] * sQ3[(k * NQF + q) * 5 + s];
        sQ2[o] = acc;
      }
      __syncthreads();
      for (int o = tid; o < NM; o += NT) {
        const int i = o / 5, s = o % 5;
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int kj = sNF[i * 3 + c];
          if (kj < 0) break;
          v += sQ2[kj * 5 + s];
        }
        out[(size_t)e * NM + o] = (mode == 0) ? -v : (-r_w[(size_t)e * NM + o] + (-v));
      }
    } else {
      for (int o = tid; o < NX; o += NT) {
        const int k = o / (NFN * 5), j = (o / 5) % NFN, s = o % 5;
        double a = 0.0, b = 0.0;
#pragma unroll 4
        for (int q = 0; q < NQF; ++q) {
          const double fp = sFP[q * D::FS + j];
          a += fp * sQ3[(k * NQF + q) * 5 + s];
          if (use_b) b += fp * sQ4[(k * NQF + q) * 5 + s];
        }
        atomicAdd(&out[((size_t)mt[k] * NFN + mt[4 + k * NFN + j]) * 5 + s], b + a);
      }
    }
    // metadata of e+2G lands in the slot freed two iterations ago
    if (e2 < g.E) {
#pragma unroll
      for (int c = 0; c < FP::MPT; ++c) {
        const int i = tid + c * NT;
        if (i < META + 4) meta_store(s2, i, rMi[c], rMd[c]);
      }
    }
  }
}

// K4 (apply): z_f = P_f^-1 r_f, column-major GEMV per face
template <int P, int NT>
__global__ void __launch_bounds__(NT)
k_precond_apply(int F, const double* __restrict__ pinv, const double* __restrict__ r,
                double* __restrict__ z) {
  constexpr int NB = Dims<P>::NB;
  __shared__ double sR[NB];
  for (int f = blockIdx.x; f < F; f += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < NB; i += NT) sR[i] = r[(size_t)f * NB + i];
    __syncthreads();
    const double* A = pinv + (size_t)f * NB * NB;
    for (int row = threadIdx.x; row < NB; row += NT) {
      double acc0 = 0.0, acc1 = 0.0;
      int c = 0;
      for (; c + 1 < NB; c += 2) {
        acc0 += A[(size_t)c * NB + row] * sR[c];
        acc1 += A[(size_t)(c + 1) * NB + row] * sR[c + 1];
      }
      if (c < NB) acc0 += A[(size_t)c * NB + row] * sR[c];
      z[(size_t)f * NB + row] = acc0 + acc1;
    }
  }
}

// ===========================================================================
// pointwise helpers and monitors
// ===========================================================================
template <int P, int NT>
__global__ void __launch_bounds__(NT)
k_volume_states(Geo g, const double* __restrict__ w, double* __restrict__ out,
                unsigned long long* status) {
  using D = Dims<P>;
  __shared__ double sPhi[D::NQ * D::NN];
  __shared__ double sW[D::NN * 5];
  for (int i = threadIdx.x; i < D::NQ * D::NN; i += NT)
    sPhi[i] = g.B[(i / D::NN) * 4 * D::NN + 3 * D::NN + i % D::NN];
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < D::NN * 5; i += NT) sW[i] = w[(size_t)e * D::NN * 5 + i];
    __syncthreads();
    for (int q = threadIdx.x; q < D::NQ; q += NT) {
      double wq[5] = {0, 0, 0, 0, 0};
      for (int i = 0; i < D::NN; ++i) {
        const double ph = sPhi[q * D::NN + i];
#pragma unroll
        for (int s = 0; s < 5; ++s) wq[s] += ph * sW[i * 5 + s];
      }
      double u[5];
      if (!to_conservative(wq, g.form, g.gamma, u)) report(status, 0, 0, e);
#pragma unroll
      for (int s = 0; s < 5; ++s) out[((size_t)e * D::NQ + q) * 5 + s] = u[s];
    }
  }
}

// monitors: per-block partial sums of the five integrals (assembly.py:595-620)
template <int P, int NT>
__global__ void __launch_bounds__(NT)
k_integrals(Geo g, const double* __restrict__ w, double* __restrict__ partial) {
  using D = Dims<P>;
  __shared__ double sPhi[D::NQ * D::NN];
  __shared__ double sW[D::NN * 5];
  __shared__ double red[5][NT];
  for (int i = threadIdx.x; i < D::NQ * D::NN; i += NT)
    sPhi[i] = g.B[(i / D::NN) * 4 * D::NN + 3 * D::NN + i % D::NN];
  double acc[5] = {0, 0, 0, 0, 0};
  const double gam = g.gamma;
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < D::NN * 5; i += NT) sW[i] = w[(size_t)e * D::NN * 5 + i];
    __syncthreads();
    for (int q = threadIdx.x; q < D::NQ; q += NT) {
      double wq[5] = {0, 0, 0, 0, 0};
      for (int i = 0; i < D::NN; ++i) {
        const double ph = sPhi[q * D::NN + i];
#pragma unroll
        for (int s = 0; s < 5; ++s) wq[s] += ph * sW[i * 5 + s];
      }
      double u[5];
      to_conservative(wq, g.form, gam, u);
      double rho, vel[3], p;
      primitive(u, gam, rho, vel, p);
      const double vw = g.qw[q] * g.det[e];
      const double sp = ::log(p) - gam * ::log(rho);
      acc[0] += vw * (-rho * sp / (gam - 1.0));
      acc[1] += vw * rho * sp;
      acc[2] += vw * 0.5 * rho * ((vel[0] * vel[0] + vel[1] * vel[1]) + vel[2] * vel[2]);
      acc[3] += vw * rho;
      acc[4] += vw * u[4];
    }
  }
  for (int c = 0; c < 5; ++c) red[c][threadIdx.x] = acc[c];
  __syncthreads();
  for (int sft = NT / 2; sft > 0; sft >>= 1) {
    if (threadIdx.x < sft)
      for (int c = 0; c < 5; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + sft];
    __syncthreads();
  }
  if (threadIdx.x < 5) partial[blockIdx.x * 5 + threadIdx.x] = red[threadIdx.x][0];
}

}  // namespace mhdg
