// Blocked Gauss-Jordan inverse with partial pivoting on the FP64 tensor cores.
//
// Replaces the reference's per-macro lu_factor / lu_solve of S
// (assembly.py:718-733, 943-976) by an explicit inverse, as k_gj_batched
// does, but organised as panels of 8 pivot columns:
//   1. the CTA factors the 8-column panel, one panel row per thread (warp
//      argmax + one barrier per pivot to combine the warps' candidates;
//      eager in-place Gauss-Jordan updates on the panel only);
//   2. the 8 steps compose to L = I + U P^T with U = panel - E (E: ones at
//      (p_t, t)), so every other column gets A += U R, R = the pivot rows
//      before the panel, a K = 8 GEMM done with mma.sync.m8n8k4.f64 on
//      accumulator tiles loaded from / stored to shared memory.
// Implicit pivoting (no row swaps): on exit A^-1[r][c] = Y[q[r]][q^-1[c]].
// Same pivot rule as the unblocked kernel (largest |a|, first index on
// ties); results agree with it and with LU to rounding.
#pragma once
#include "mhdg_kernels.cuh"

namespace mhdg {

// GM = true: the padded working matrix lives in a per-CTA global scratch
// slab (L2-resident) instead of shared memory, for orders whose matrix does
// not fit (N = 175 at k = 4: 248 KB); U / R / pivot candidates stay in
// shared memory.
template <int N>
struct GJB {
  static constexpr int NP = (N + 7) / 8 * 8;                 // padded order
  static constexpr int S = (NP % 16 == 0) ? NP + 8 : NP;     // A row stride = 8 (mod 16) doubles
  static constexpr int SU = NP + ((4 - NP % 16) + 16) % 16;  // U / R stride = 4 (mod 16)
  static constexpr int T = NP / 8;
  static constexpr int NPAN = (N + 7) / 8;
  static constexpr int NW = (NP + 31) / 32;                  // one panel row per thread
  static constexpr int NT = 32 * NW;
  static constexpr size_t bytes = (size_t)(NP * S + 2 * 8 * SU + 2 * NW * 10) * 8 + (size_t)(2 * N + 4) * 4;
  static constexpr size_t bytes_gm = (size_t)(2 * 8 * SU + 2 * NW * 10) * 8 + (size_t)(2 * N + 4) * 4;
  static constexpr size_t slab = (size_t)NP * S;   // doubles per CTA (GM)
};

template <int N, bool GM = false>
__global__ void __launch_bounds__(GJB<N>::NT, 2)
k_gj_blocked(int nmat, double* __restrict__ mats, unsigned long long* status, double* __restrict__ scratch = nullptr) {
  using G = GJB<N>;
  constexpr int NP = G::NP, S = G::S, SU = G::SU, T = G::T, NT = G::NT, NW = G::NW;
  extern __shared__ __align__(16) double smem[];
  double* A = GM ? scratch + (size_t)blockIdx.x * G::slab : smem;   // NP x S
  double* U = GM ? smem : A + NP * S;   // [8][SU]  (k-major)
  double* R = U + 8 * SU;           // [8][SU]
  double* cand = R + 8 * SU;        // [2][NW][10]: |a|, row index, 8 row values
  int* q = (int*)(cand + 2 * NW * 10);
  int* qi = q + N;
  int* flag = qi + N;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = tid;                // this thread's panel row
  // padding rows / columns stay zero through every update (U and R vanish there)
  for (int idx = tid; idx < NP * S; idx += NT) A[idx] = 0.0;
  for (int m = blockIdx.x; m < nmat; m += gridDim.x) {
    double* M = mats + (size_t)m * N * N;
    __syncthreads();
    if constexpr (N % 2 == 0) {   // row pairs as double2
      const double2* M2 = reinterpret_cast<const double2*>(M);
#pragma unroll 8
      for (int i = tid; i < N * N / 2; i += NT) {
        const int rr = (2 * i) / N, c = (2 * i) % N;
        *reinterpret_cast<double2*>(A + rr * S + c) = __ldcs(M2 + i);
      }
    } else {
      for (int i = tid; i < N * N; i += NT) A[(i / N) * S + i % N] = __ldcs(M + i);
    }
    bool used = r >= N;
    bool ok = true;
    __syncthreads();
    for (int pan = 0; pan < G::NPAN; ++pan) {
      const int k0 = pan * 8, nbp = min(8, N - k0);
      double pv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) pv[j] = (r < NP) ? A[r * S + k0 + j] : 0.0;
      int pt[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        pt[t] = -1;
        if (t < nbp) {
          // pivot: unused row with the largest |a_rt|, first index on ties
          // warp argmax on the bit pattern of |a| (monotone for a >= 0):
          // max of the high word (+1, so used rows = 0 lose), then of the
          // low word among the ties, then the smallest row index
          const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(pv[t]));
          const unsigned hi = used ? 0u : (unsigned)(bits >> 32) + 1u, lo = used ? 0u : (unsigned)bits;
          const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
          const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
          const int bi = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)r : 0x7fffffffu);
          double* cb = cand + ((t & 1) * NW + warp) * 10;
          if (lane == 0) {
            cb[0] = mhi == 0u ? -1.0 : __longlong_as_double((long long)(((unsigned long long)(mhi - 1u) << 32) | mlo));
            cb[1] = (double)(mhi == 0u ? N : bi);
          }
          if (r == bi) {
#pragma unroll
            for (int j = 0; j < 8; ++j) cb[2 + j] = pv[j];
          }
          __syncthreads();
          const double* c0 = cand + (t & 1) * NW * 10;
          int w = 0;
          double bv = c0[0];
          int bidx = (int)c0[1];
#pragma unroll
          for (int w2 = 1; w2 < NW; ++w2) {
            const double v = c0[w2 * 10];
            const int ix = (int)c0[w2 * 10 + 1];
            if (v > bv || (v == bv && ix < bidx)) { bv = v; bidx = ix; w = w2; }
          }
          const int p = bidx < N ? bidx : 0;
          pt[t] = p;
          double prow[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) prow[j] = c0[w * 10 + 2 + j];
          const double piv = prow[t];
          if (!(fabs(piv) > 0.0) || !isfinite(piv)) ok = false;
          const double pinv = 1.0 / piv;
#pragma unroll
          for (int j = 0; j < 8; ++j) prow[j] = (j == t ? 1.0 : prow[j]) * pinv;
          const bool isp = r == p;
          const double cr = pv[t];
          used = used || isp;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double v = (j == t ? 0.0 : pv[j]) - cr * prow[j];
            pv[j] = isp ? prow[j] : v;
          }
        }
      }
      if (tid == 0)
        for (int t = 0; t < nbp; ++t) q[k0 + t] = pt[t];
      // panel final values, U = panel - E, R = pivot rows outside the panel
      if (r < NP) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          A[r * S + k0 + j] = pv[j];
          U[j * SU + r] = (pt[j] >= 0) ? pv[j] - (r == pt[j] ? 1.0 : 0.0) : 0.0;
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t)
        for (int c = tid; c < NP; c += NT)
          R[t * SU + c] = (pt[t] >= 0 && (c < k0 || c >= k0 + 8)) ? A[pt[t] * S + c] : 0.0;
      __syncthreads();
      // rank-8 update of all other column tiles on the tensor cores
      for (int mi = warp; mi < T; mi += NW) {
        const int kk0 = lane & 3, row = mi * 8 + (lane >> 2);
        const double a0 = U[kk0 * SU + row], a1 = U[(kk0 + 4) * SU + row];
        double* cp = A + row * S + (lane & 3) * 2;
        const double* rp = R + kk0 * SU + (lane >> 2);
#pragma unroll 4
        for (int ni = 0; ni < T; ++ni) {
          if (ni == pan) continue;
          const double2 cv = *reinterpret_cast<const double2*>(cp + ni * 8);
          double c[2] = {cv.x, cv.y};
          dmma_8x8x4(c, a0, rp[ni * 8]);
          dmma_8x8x4(c, a1, rp[4 * SU + ni * 8]);
          *reinterpret_cast<double2*>(cp + ni * 8) = make_double2(c[0], c[1]);
        }
      }
      __syncthreads();
    }
    for (int k = tid; k < N; k += NT) qi[q[k]] = k;
    __syncthreads();
    int bad = !ok;
    if constexpr (N % 2 == 0) {
      double2* M2 = reinterpret_cast<double2*>(M);
#pragma unroll 4
      for (int i = tid; i < N * N / 2; i += NT) {
        const int c = (2 * i) / N, rr = (2 * i) % N, qc = qi[c];
        const double v0 = A[q[rr] * S + qc], v1 = A[q[rr + 1] * S + qc];
        bad |= !isfinite(v0) || !isfinite(v1);
        M2[i] = make_double2(v0, v1);
      }
    } else {
      for (int i = tid; i < N * N; i += NT) {
        const double v = A[q[i % N] * S + qi[i / N]];
        bad |= !isfinite(v);
        M[i] = v;
      }
    }
    if (__syncthreads_or(bad) && tid == 0) report(status, 0, 0, m);
  }
}

}  // namespace mhdg
