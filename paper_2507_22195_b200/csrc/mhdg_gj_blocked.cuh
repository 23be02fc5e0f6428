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

namespace mhdg {

// ===========================================================================
// Gauss-Jordan inverse with one-panel lookahead (k_gj_la2).
//
// Same arithmetic as k_gj_blocked (8-column panels, implicit partial
// pivoting, composite panel transform A += U R on the FP64 tensor cores) but
// the serial pivot search no longer stops the whole CTA at a barrier per
// pivot: the panel warps factor panel p + 1 while the update warps apply
// panel p's update to every other column.  Between two CTA barriers:
//   panel warps : R_p on panel p+1's columns, A[:, p+1] += U_p R_p, factor
//                 panel p+1 -> U_{p+1} (double-buffered), pivots
//   update warps: A[:, c] += U_p R_p[:, c] on their own column tiles (all but
//                 panels p, p+1), R_p read straight from the pivot rows
// Panel p+1's columns therefore hold every update < p+1 when it is factored,
// and no two warps touch the same column in one interval.
//
// With NPW panel warps the panel rows are split over
// NPW warps (rows 32 (pw + NPW i) + lane), so each pivot step handles
// RPL = NP / (32 NPW) rows per lane; the warps' argmax candidates and the
// pivot row meet in shared memory behind a named barrier of the panel
// warps.  A pivot step's dependent chain shortens with the rows per lane
// (measured ~1100 cycles at 4 rows / lane, ~480 at 2).
// ===========================================================================
#ifndef MHDG_GJ_STRIDE2
#define MHDG_GJ_STRIDE2 0   // measured slower (18.57 vs 18.42 ms): the C-tile accesses lose more
#endif
template <int N, int NWT, int NPW>
struct GJLA2 {
  using G = GJB<N>;
  // row stride S = 2 (mod 4) doubles: the panel warps' row-per-lane loads /
  // stores and the permuted gathers then spread over 8 bank pairs instead of
  // the 2 of a stride = 8 (mod 16); even, so the double2 C tiles stay aligned
#if MHDG_GJ_STRIDE2
  static constexpr int NP = G::NP, S = G::NP + 2, T = G::T, NPAN = G::NPAN;
#else
  static constexpr int NP = G::NP, S = G::S, T = G::T, NPAN = G::NPAN;
#endif
  static constexpr int RPL = (NP + 32 * NPW - 1) / (32 * NPW);
  static constexpr int NT = 32 * NWT;
  static constexpr int UF = T * 2 * 32;
  static constexpr int XD = NPW > 1 ? 64 : 16;   // pivot-row / diagonal-block exchange (doubles)
  static constexpr size_t bytes = (size_t)(NP * S + 2 * UF + XD + 2 * NPW) * 8 + (size_t)(2 * NP + 4 + 2 * NPW) * 4;
  static constexpr size_t bytes_ga = (size_t)(2 * UF + XD + 2 * NPW) * 8 + (size_t)(2 * NP + 4 + 2 * NPW) * 4;
  static constexpr size_t slab = (size_t)NP * S;   // doubles per CTA (GA)
};

#ifndef MHDG_GJ_TILE_STORE
#define MHDG_GJ_TILE_STORE 1
#endif
#ifndef MHDG_GJ_FASTRCP
#define MHDG_GJ_FASTRCP 1
#endif
#ifndef MHDG_GJ_MINB_SMALL
#define MHDG_GJ_MINB_SMALL 6   // face blocks: 6 CTAs / SM (measured best)
#endif
// Matrix sources for the lookahead Gauss-Jordan: load(m, A, S, ...) fills the
// N x N block of working matrix A (row stride S, padding untouched) for item
// m; every thread of the CTA calls it.  The inverse is written to mats[m].
template <int N>
struct GjGlobalSrc {   // the matrix is read from mats[m] and overwritten
  static constexpr size_t extra_bytes = 0;
  const double* mats;
  __device__ __forceinline__ void init(double*, int, int) const {}
  // the next matrix towards L2 while this one is inverted
  __device__ __forceinline__ void prefetch(int m, int tid, int NT) const {
    const char* M = reinterpret_cast<const char*>(mats + (size_t)m * N * N);
    for (int i = tid * 128; i < N * N * 8; i += NT * 128) prefetch_l2(M + i);
  }
  __device__ __forceinline__ void load(int m, double* A, int S, double*, double*, int tid, int NT) const {
    const double* M = mats + (size_t)m * N * N;
    if constexpr (N % 2 == 0) {
      const double2* M2 = reinterpret_cast<const double2*>(M);
      for (int i = tid; i < N * N / 2; i += NT) {
        const int rr = (2 * i) / N, c = (2 * i) % N;
        *reinterpret_cast<double2*>(A + rr * S + c) = __ldcs(M2 + i);
      }
    } else {
      for (int i = tid; i < N * N; i += NT) A[(i / N) * S + i % N] = __ldcs(M + i);
    }
  }
};

// Matrix selection and the diagonal-pivot pass (GjPass): with nopiv the
// pivots are taken on the diagonal (no search on the pivot chain: a pivot
// step is broadcast -> reciprocal -> update); every panel warp checks, off
// the chain, that the pivot is at least GJ_TAU times the largest remaining
// entry of its rows in that column.  A matrix that fails the check (or meets
// a zero / non-finite pivot) is left untouched in `mats` and appended to
// fb_list; the partial-pivoting pass then runs over that list (list /
// count_dev), so singular blocks are still detected and reported by the
// pivoting elimination exactly as before.
#ifndef MHDG_GJ_TAU
#define MHDG_GJ_TAU 0.05
#endif
#ifndef MHDG_GJ_PREFETCH
#define MHDG_GJ_PREFETCH 1   // L2 prefetch of the next matrix / face rows
#endif
#ifndef MHDG_GJ_SCHED_ROLES
#define MHDG_GJ_SCHED_ROLES 0   // panel warps = the warps on hardware scheduler 0
#endif
#ifndef MHDG_GJ_BLOCKPANEL
#define MHDG_GJ_BLOCKPANEL 1   // diagonal-pivot pass: panels through the 8 x 8 block inverse
#endif
struct GjPass {
  const int* list;       // matrices to process (nullptr: 0 .. nmat-1)
  const int* count_dev;  // length of list (device), when list != nullptr
  int* fb_count;         // nopiv pass: fallback list length
  int* fb_list;          // nopiv pass: fallback matrix ids
  double* slab = nullptr;   // GA: per-CTA global working matrices (NP x S each)
};

// GA: the working matrix lives in a per-CTA global slab (L2-resident) instead
// of shared memory, for orders whose matrix does not fit (k = 4: N = 175,
// 259 KB); the U panels, pivot data and everything else stay in shared
// memory.  Within one SM the global accesses of the CTA's warps are coherent
// through L1 after the CTA barriers.
template <int N, int NWT, int NPW, class Src, bool NOPIV = false, bool GA = false>
__device__ __forceinline__ void gj_la2_body(int nmat, double* __restrict__ mats, unsigned long long* status,
                                            const Src& src, GjPass pass = GjPass{nullptr, nullptr, nullptr, nullptr}) {
  using L = GJLA2<N, NWT, NPW>;
  constexpr int NP = L::NP, S = L::S, T = L::T, NPAN = L::NPAN, RPL = L::RPL, NT = L::NT;
  extern __shared__ __align__(16) double smem[];
  double* A = GA ? pass.slab + (size_t)blockIdx.x * NP * S : smem;   // NP x S
  double* Ub = GA ? smem : A + NP * S;     // 2 x UF
  double* sProw = Ub + 2 * L::UF;          // 2 x 8: pivot row of the current step (block panels: 8 x 8 diagonal block)
  unsigned* sCand = reinterpret_cast<unsigned*>(sProw + L::XD);  // [NPW][3]: hi, lo, row
  int* q = (int*)(sCand + 4 * NPW);        // NP: pivot row of step k
  int* qi = q + NP;
  int* flag = qi + NP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kq = lane & 3, nr = lane >> 2;
  // Warp roles by hardware scheduler.  A warp issues on scheduler
  // %warpid % 4 (measured: a dependent DFMA chain sharing a scheduler with
  // a DMMA stream slows from 8.8 to 47.5 cycles per operation, a chain on
  // another scheduler is unaffected; the second co-resident CTA's warps sit
  // one scheduler further, so the warp index alone does not tell).  When
  // the CTA has NPW warps on hardware scheduler 0 they become the panel
  // warps, so the serial panel chains of all co-resident CTAs share one
  // scheduler and the update warps' DMMA streams run on the other three;
  // otherwise the first NPW warps are the panel warps.
  bool panel = warp < NPW;
  int pw = warp, n_panel_below = min(NPW, warp);
  if constexpr (4 * NPW <= NWT && MHDG_GJ_SCHED_ROLES) {
    unsigned hw;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(hw));
    if (lane == 0) q[warp] = (int)(hw & 3u);
    __syncthreads();
    int cnt0 = 0, mine = 0, below = 0;
#pragma unroll
    for (int w2 = 0; w2 < NWT; ++w2) {
      const bool p2 = q[w2] == 0 && cnt0 < NPW;
      if (w2 == warp) { mine = p2 ? cnt0 : -1; }
      if (p2) {
        ++cnt0;
        if (w2 < warp) ++below;
      }
    }
    if (cnt0 == NPW) {
      panel = mine >= 0;
      pw = mine >= 0 ? mine : 0;
      n_panel_below = below;
    }
    __syncthreads();
  }
  auto psync = [&]() {
    if (NPW > 1) asm volatile("bar.sync 1, %0;" ::"r"(32 * NPW) : "memory");
    else __syncwarp();
  };
  for (int idx = tid; idx < NP * S; idx += NT) A[idx] = 0.0;

  auto row_of = [&](int i) { return 32 * (pw + NPW * i) + lane; };
  auto factor_panel = [&](int pan, unsigned& used, bool& ok) {
    const int k0 = pan * 8, nbp = min(8, N - k0);
    double a[RPL][8];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = row_of(i);
#pragma unroll
      for (int j = 0; j < 8; ++j) a[i][j] = r < NP ? A[r * S + k0 + j] : 0.0;
    }
    int pt[8];
    if constexpr (NOPIV) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        pt[t] = -1;
        if (t < nbp) {
          const int p = k0 + t;
          // ratio check, off the pivot chain: largest |a_rt| over this warp's
          // rows r > p (hi word of the bit pattern: a bound within 2^-20)
          unsigned bhi = 0u;
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int r = row_of(i);
            const unsigned hi = (unsigned)((unsigned long long)__double_as_longlong(fabs(a[i][t])) >> 32);
            if (r < N && r > p && hi > bhi) bhi = hi;
          }
          const unsigned mhi = __reduce_max_sync(0xffffffffu, bhi);
          pt[t] = p;
          if (pw == 0 && lane == 0) q[p] = p;
          const int owner = p & 31, oslot = (p >> 5) / NPW, ow = (p >> 5) % NPW;
          double prow[8];
          if (NPW > 1) {
            double* pr = sProw + (t & 1) * 8;   // double-buffered across pivots
            if (pw == ow && lane == owner)
#pragma unroll
              for (int i = 0; i < RPL; ++i)
                if (i == oslot)
#pragma unroll
                  for (int j = 0; j < 8; ++j) pr[j] = a[i][j];
            psync();
#pragma unroll
            for (int j = 0; j < 8; ++j) prow[j] = pr[j];
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              double v = a[0][j];
#pragma unroll
              for (int i = 1; i < RPL; ++i) v = oslot == i ? a[i][j] : v;
              prow[j] = __shfl_sync(0xffffffffu, v, owner);
            }
          }
          const double piv = prow[t];
          const double cmax = __longlong_as_double((long long)((unsigned long long)mhi << 32));
          if (!(fabs(piv) > 0.0) || !isfinite(piv) || fabs(piv) < MHDG_GJ_TAU * cmax) ok = false;
          const double pinv = drcp(piv);
#pragma unroll
          for (int j = 0; j < 8; ++j) prow[j] = (j == t ? 1.0 : prow[j]) * pinv;
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const bool isp = (pw == ow) && (lane == owner) && (oslot == i);
            const double cr = a[i][t];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const double v = (j == t ? 0.0 : a[i][j]) - cr * prow[j];
              a[i][j] = isp ? prow[j] : v;
            }
          }
        }
      }
    } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      pt[t] = -1;
      if (t < nbp) {
        unsigned bhi = 0u, blo = 0u;
        int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const int r = row_of(i);
          const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(a[i][t]));
          const bool cand = r < N && !((used >> i) & 1u);
          const unsigned hi = cand ? (unsigned)(bits >> 32) + 1u : 0u, lo = cand ? (unsigned)bits : 0u;
          if (hi > bhi || (hi == bhi && lo > blo)) { bhi = hi; blo = lo; bi = r; }
        }
        // warp argmax: largest (hi, lo), smallest row on ties
        const unsigned mhi = __reduce_max_sync(0xffffffffu, bhi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, bhi == mhi ? blo : 0u);
        const int wp = (int)__reduce_min_sync(0xffffffffu, (bhi == mhi && blo == mlo) ? (unsigned)bi : 0x7fffffffu);
        int p = wp;
        if (NPW > 1) {
          if (lane == 0) {
            sCand[pw * 3 + 0] = mhi;
            sCand[pw * 3 + 1] = mlo;
            sCand[pw * 3 + 2] = (unsigned)wp;
          }
          psync();
          unsigned ghi = sCand[0], glo = sCand[1];
          p = (int)sCand[2];
#pragma unroll
          for (int w2 = 1; w2 < NPW; ++w2) {
            const unsigned h2 = sCand[w2 * 3], l2 = sCand[w2 * 3 + 1];
            const int r2 = (int)sCand[w2 * 3 + 2];
            if (h2 > ghi || (h2 == ghi && (l2 > glo || (l2 == glo && r2 < p)))) { ghi = h2; glo = l2; p = r2; }
          }
          if (ghi == 0u) p = 0x7fffffff;
        } else if (mhi == 0u) {
          p = 0x7fffffff;
        }
        if (p >= N) { ok = false; p = 0; }
        pt[t] = p;
        if (pw == 0 && lane == 0) q[k0 + t] = p;
        const int owner = p & 31, oslot = (p >> 5) / NPW, ow = (p >> 5) % NPW;
        double prow[8];
        if (NPW > 1) {
          if (pw == ow && lane == owner)
#pragma unroll
            for (int i = 0; i < RPL; ++i)
              if (i == oslot)
#pragma unroll
                for (int j = 0; j < 8; ++j) sProw[j] = a[i][j];
          psync();
#pragma unroll
          for (int j = 0; j < 8; ++j) prow[j] = sProw[j];
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            double v = a[0][j];
#pragma unroll
            for (int i = 1; i < RPL; ++i) v = oslot == i ? a[i][j] : v;
            prow[j] = __shfl_sync(0xffffffffu, v, owner);
          }
        }
        const double piv = prow[t];
        if (!(fabs(piv) > 0.0) || !isfinite(piv)) ok = false;
        #if MHDG_GJ_FASTRCP
        const double pinv = drcp(piv);   // branch-free reciprocal on the pivot chain
#else
        const double pinv = 1.0 / piv;
#endif
#pragma unroll
        for (int j = 0; j < 8; ++j) prow[j] = (j == t ? 1.0 : prow[j]) * pinv;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const bool isp = (pw == ow) && (lane == owner) && (oslot == i);
          const double cr = a[i][t];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double v = (j == t ? 0.0 : a[i][j]) - cr * prow[j];
            a[i][j] = isp ? prow[j] : v;
          }
          if (isp) used |= 1u << i;
        }
      }
    }
    }
    double* U = Ub + (pan & 1) * L::UF;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = row_of(i);
      if (r < NP) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          A[r * S + k0 + j] = a[i][j];
          const double u = (pt[j] >= 0) ? a[i][j] - (r == pt[j] ? 1.0 : 0.0) : 0.0;
          U[((r >> 3) * 2 + (j >> 2)) * 32 + (r & 7) * 4 + (j & 3)] = u;
        }
      }
    }
    if (pw == 0 && lane == 0)
      for (int t = nbp; t < 8; ++t) q[k0 + t] = -1;
  };

  // Diagonal-pivot pass, block form (MHDG_GJ_BLOCKPANEL).  The eight Gauss-
  // Jordan steps of panel p with pivots on its own diagonal block D_p compose
  // to  panel <- [ G_p = D_p^-1 on the block rows ; -P G_p elsewhere ],  and
  // D_{p+1} needs, of panel p's whole update, one tile:
  //   D_{p+1} = A[p+1][p+1] + U_p[p+1] R_p[p+1],  U_p = panel_p - E.
  // So the serial chain is  one tile update -> 8 x 8 inverse  per panel, on
  // ONE warp (the chain warp), and everything else is throughput work:
  //   phase 1 (all warps)   : panel p's columns <- -P G_p, U_p fragments;
  //                           the R tile the chain needs next is copied aside
  //   phase 2 (chain warp)  : D_{p+1}, G_{p+1} = D_{p+1}^-1 (cooperative in
  //                           the C-fragment layout: row lane / 4, columns
  //                           2 (lane % 4), +1; shuffles only, and the next
  //                           pivot's reciprocal is started one step ahead)
  //           (update warps): A[:, c] += U_p R_p[c] for every column tile
  //                           c != p (tile (p+1, p+1) excepted: the chain's)
  // Checks, lane-local and branch-free: every in-block pivot is at least
  // GJ_TAU times the entries below it in D, and no composite multiplier
  // (-P G below the block) exceeds 1 / GJ_TAU; a matrix failing either goes
  // to the partial-pivoting pass.
  double* sG = Ub + L::UF;   // G row-major 8 x 8 (the second U buffer is free in this pass)
  double* sR = sG + 64;      // R_p on panel p+1's columns, row-major 8 x 8
  static_assert(!(NOPIV && MHDG_GJ_BLOCKPANEL) || L::UF >= 128, "block-panel scratch");
#ifdef MHDG_RES_TIMING
  long long tp = 0;
#define BP_T0() tp = clock64()
#define BP_T(k, cond) do { const long long t_ = clock64(); if (cond) atomicAdd(&g_res_clk[(N == 100 ? 16 : 21) + (k)], (unsigned long long)(t_ - tp)); tp = t_; } while (0)
#else
#define BP_T0() do { } while (0)
#define BP_T(k, cond) do { } while (0)
#endif
  // phase 1: the panel transform of panel pn, all warps
  auto panel_transform = [&](int pn, bool& ok) {
    const int k0n = pn * 8, nbp = min(8, N - k0n);
    const double b0 = sG[kq * 8 + nr], b1 = sG[(kq + 4) * 8 + nr];
    const double2 gd = *reinterpret_cast<const double2*>(sG + nr * 8 + 2 * kq);
    int nbad = 0;
#pragma unroll 2
    for (int rt = warp; rt < T; rt += NWT) {
      const double* ap = A + (rt * 8 + nr) * S + k0n + kq;
      double c[2] = {0.0, 0.0};
      dmma_8x8x4(c, ap[0], b0);
      dmma_8x8x4(c, ap[4], b1);
      __syncwarp();   // the tile's A fragments are read before its columns are rewritten
      double n0 = -c[0], n1 = -c[1];
      nbad |= (int)(rt > pn) & ((int)!(fabs(n0) <= 1.0 / MHDG_GJ_TAU) | (int)!(fabs(n1) <= 1.0 / MHDG_GJ_TAU));
      double u0 = n0, u1 = n1;
      if (rt == pn) {
        n0 = gd.x;
        n1 = gd.y;
        u0 = gd.x - ((nr == 2 * kq && nr < nbp) ? 1.0 : 0.0);
        u1 = gd.y - ((nr == 2 * kq + 1 && nr < nbp) ? 1.0 : 0.0);
      }
      *reinterpret_cast<double2*>(A + (rt * 8 + nr) * S + k0n + kq * 2) = make_double2(n0, n1);
      *reinterpret_cast<double2*>(Ub + (rt * 2 + (kq >> 1)) * 32 + nr * 4 + 2 * (kq & 1)) = make_double2(u0, u1);
    }
    // the R tile of the next panel's columns, for the chain warp (the owner
    // of that column tile rewrites it during phase 2)
    if (warp == NWT - 1 && pn + 1 < T)
      *reinterpret_cast<double2*>(sR + nr * 8 + 2 * kq) =
          *reinterpret_cast<const double2*>(A + (k0n + nr) * S + k0n + 8 + 2 * kq);
    if (__any_sync(0xffffffffu, nbad) && lane == 0) *flag = 1;
  };
  // phase 2, chain warp: D_pn (with panel pn-1's update when Up) and G_pn
  auto chain_block = [&](int pn, bool with_update, bool& ok) {
    const int k0n = pn * 8, nbp = min(8, N - k0n);
    BP_T0();
    double d0, d1;
    {
      const double2 dd = *reinterpret_cast<const double2*>(A + (k0n + nr) * S + k0n + kq * 2);
      double c[2] = {dd.x, dd.y};
      if (with_update) {
        dmma_8x8x4(c, Ub[(pn * 2 + 0) * 32 + lane], sR[kq * 8 + nr]);
        dmma_8x8x4(c, Ub[(pn * 2 + 1) * 32 + lane], sR[(kq + 4) * 8 + nr]);
      }
      d0 = c[0];
      d1 = c[1];
    }
    BP_T(0, lane == 0);
    int nbad = 0;
    double piv = __shfl_sync(0xffffffffu, d0, 0);
    double pinv = drcp(piv);
#pragma unroll 1
    for (int t = 0; t < nbp; ++t) {
      const double dt = (t & 1) ? d1 : d0, dn = (t & 1) ? d0 : d1;   // column t / t + 1 slots
      const double p0 = __shfl_sync(0xffffffffu, d0, t * 4 + kq);
      const double p1 = __shfl_sync(0xffffffffu, d1, t * 4 + kq);
      const double cr = __shfl_sync(0xffffffffu, dt, (lane & ~3) | (t >> 1));
      // next pivot one step ahead: D[t+1][t+1] - D[t+1][t] (D[t][t+1] pinv),
      // the same operations its owner lane performs below
      const int t1 = (t + 1) & 7;
      const double la = __shfl_sync(0xffffffffu, dn, t1 * 4 + (t1 >> 1));
      const double lb = __shfl_sync(0xffffffffu, dt, t1 * 4 + (t >> 1));
      const double lc = __shfl_sync(0xffffffffu, dn, t * 4 + (t1 >> 1));
      const double apiv = fabs(piv);
      nbad |= (int)!(apiv > 0.0) | (int)!(apiv < 1.7976931348623157e308) |
              ((int)(nr > t) & (int)(apiv < MHDG_GJ_TAU * fabs(cr)));
      const double pnext = la - lb * (lc * pinv);
      const double pinv_next = drcp(pnext);
      const bool c0t = 2 * kq == t, c1t = 2 * kq + 1 == t;
      const double s0 = (c0t ? 1.0 : p0) * pinv, s1 = (c1t ? 1.0 : p1) * pinv;
      const double v0 = (c0t ? 0.0 : d0) - cr * s0, v1 = (c1t ? 0.0 : d1) - cr * s1;
      d0 = nr == t ? s0 : v0;
      d1 = nr == t ? s1 : v1;
      piv = pnext;
      pinv = pinv_next;
    }
    BP_T(1, lane == 0);
    if (lane < 8) q[k0n + lane] = lane < nbp ? k0n + lane : -1;
    *reinterpret_cast<double2*>(sG + nr * 8 + 2 * kq) = make_double2(d0, d1);
    if (__any_sync(0xffffffffu, nbad) && lane == 0) *flag = 1;
    (void)ok;
    BP_T(2, lane == 0);
  };

  auto update_tile = [&](const double* U, int ct, double r0, double r1, int rt0, int rt1, int rts) {
    for (int rt = rt0; rt < rt1; rt += rts) {
      double* cp = A + (rt * 8 + nr) * S + ct * 8 + kq * 2;
      const double2 cv = *reinterpret_cast<const double2*>(cp);
      double c[2] = {cv.x, cv.y};
      dmma_8x8x4(c, U[(rt * 2 + 0) * 32 + lane], r0);
      dmma_8x8x4(c, U[(rt * 2 + 1) * 32 + lane], r1);
      *reinterpret_cast<double2*>(cp) = make_double2(c[0], c[1]);
    }
  };

  double* ex = smem + ((GA ? L::bytes_ga : L::bytes) + 15) / 16 * 2;   // the source's scratch
  src.init(ex, tid, NT);
  if (pass.list) nmat = *pass.count_dev;
  for (int mi = blockIdx.x; mi < nmat; mi += gridDim.x) {
    const int m = pass.list ? pass.list[mi] : mi;
    double* M = mats + (size_t)m * N * N;
    __syncthreads();
#ifdef MHDG_RES_TIMING
    // experiment builds: [b] load, [b+1] panel-warp busy, [b+2] update-warp
    // busy, [b+3] interval total, [b+4] store (b = 5: order 100, 10: others)
    constexpr int TB = (N == 100) ? 5 : 10;
    long long tg = clock64();
#define GJ_T(k, cond) do { const long long t_ = clock64(); if (cond) atomicAdd(&g_res_clk[TB + (k)], (unsigned long long)(t_ - tg)); } while (0)
#define GJ_T0() tg = clock64()
#else
#define GJ_T(k, cond) do { } while (0)
#define GJ_T0() do { } while (0)
#endif
    src.load(m, A, S, ex, Ub, tid, NT);   // Ub is free until the first panel
    if (MHDG_GJ_PREFETCH && mi + (int)gridDim.x < nmat) src.prefetch(pass.list ? pass.list[mi + gridDim.x] : mi + (int)gridDim.x, tid, NT);
    if (tid == 0) *flag = 0;
    __syncthreads();
    GJ_T(0, tid == 0);
    unsigned used = 0u;
    bool ok = true;
    for (int pan = -1; pan < NPAN; ++pan) {
      GJ_T0();
      const double* U = Ub + (pan & 1) * L::UF;
      const int k0 = pan * 8, nxt = pan + 1;
      constexpr bool BP = NOPIV && MHDG_GJ_BLOCKPANEL;
      if constexpr (BP) {
        U = Ub;
        if (pan >= 0) {
          panel_transform(pan, ok);
          __syncthreads();
          GJ_T(1, tid == 0);   // timing builds: phase 1 in the "panel busy" slot
          GJ_T0();
        }
      }
      if (BP && panel) {
        if constexpr (BP)
          if (pw == 0 && nxt < NPAN) chain_block(nxt, pan >= 0, ok);
      } else if (pan < 0) {
        if constexpr (!BP)
          if (panel) factor_panel(0, used, ok);
      } else if (panel) {
        if (!BP && nxt < NPAN) {
          // R_p on panel p+1's columns (read by all panel warps before any
          // of them updates those columns), update them, factor panel p+1
          const int c = nxt * 8 + nr;
          const double r0 = q[k0 + kq] >= 0 ? A[q[k0 + kq] * S + c] : 0.0;
          const double r1 = q[k0 + kq + 4] >= 0 ? A[q[k0 + kq + 4] * S + c] : 0.0;
          psync();
          update_tile(U, nxt, r0, r1, pw, T, NPW);
          psync();
          factor_panel(nxt, used, ok);
        }
      } else {
        const int uw = warp - n_panel_below, nuw = NWT - NPW;
        const int pr0 = q[k0 + kq], pr1 = q[k0 + kq + 4];
#ifndef MHDG_GJ_UREG
#define MHDG_GJ_UREG 1
#endif
#if MHDG_GJ_UREG
        // the panel's U fragments stay in registers across this warp's
        // column tiles (they were re-read from shared memory per tile: the
        // update loop is shared-memory-bandwidth bound)
        double u0[T], u1[T];
#pragma unroll
        for (int rt = 0; rt < T; ++rt) {
          u0[rt] = U[(rt * 2 + 0) * 32 + lane];
          u1[rt] = U[(rt * 2 + 1) * 32 + lane];
        }
#endif
        int slot = 0;
        for (int ct = 0; ct < T; ++ct) {
          if (ct == pan || (!BP && ct == nxt)) continue;
          if ((slot++ % nuw) != uw) continue;
          const int c = ct * 8 + nr;
          const double r0 = pr0 >= 0 ? A[pr0 * S + c] : 0.0;
          const double r1 = pr1 >= 0 ? A[pr1 * S + c] : 0.0;
          __syncwarp();
#if MHDG_GJ_UREG
#pragma unroll
          for (int rt = 0; rt < T; ++rt) {
            if (BP && ct == nxt && rt == nxt) continue;   // the chain warp's tile
            double* cp = A + (rt * 8 + nr) * S + ct * 8 + kq * 2;
            const double2 cv = *reinterpret_cast<const double2*>(cp);
            double cc[2] = {cv.x, cv.y};
            dmma_8x8x4(cc, u0[rt], r0);
            dmma_8x8x4(cc, u1[rt], r1);
            *reinterpret_cast<double2*>(cp) = make_double2(cc[0], cc[1]);
          }
#else
          update_tile(U, ct, r0, r1, 0, T, 1);
#endif
        }
      }
      if (!BP) GJ_T(1, panel && pw == 0 && lane == 0);
      GJ_T(2, !panel && warp - n_panel_below == 0 && lane == 0);
      __syncthreads();
      GJ_T(3, tid == 0);
    }
    GJ_T0();
    if (panel && __any_sync(0xffffffffu, !ok) && lane == 0) *flag = 1;
    for (int k = tid; k < N; k += NT) qi[q[k]] = k;
    __syncthreads();
    int bad = *flag;
    if constexpr (NOPIV) {
      if (bad) {   // leave S in place for the pivoting pass
        if (tid == 0) pass.fb_list[atomicAdd(pass.fb_count, 1)] = m;
        continue;
      }
    }
#if MHDG_GJ_TILE_STORE
    // column-major inverse in 4-row x 8-column tiles per warp: the gathered
    // rows q[r] / columns qi[c] spread over the banks (a column walk hits
    // only the two bank pairs of the row stride S = 8 mod 16), and each
    // column's 4 rows are one 32-byte sector of the output
    {
      constexpr int RT = (N + 3) / 4, CT = (N + 7) / 8;
      const int r4 = lane & 3, c8 = lane >> 2;
      for (int t = warp; t < RT * CT; t += NT / 32) {
        const int r = (t % RT) * 4 + r4, c = (t / RT) * 8 + c8;
        if (r < N && c < N) {
          const double v = A[q[r] * S + qi[c]];
          bad |= !isfinite(v);
          M[(size_t)c * N + r] = v;
        }
      }
    }
#else
    if constexpr (N % 2 == 0) {
      double2* M2 = reinterpret_cast<double2*>(M);
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
#endif
    GJ_T(4, tid == 0);
    if (__syncthreads_or(bad) && tid == 0) report(status, 0, 0, m);
  }
}

template <int N, int NWT, int NPW, bool NOPIV = false, bool GA = false>
__global__ void __launch_bounds__(GJLA2<N, NWT, NPW>::NT, (N < 64 ? MHDG_GJ_MINB_SMALL : 2))
k_gj_la2(int nmat, double* __restrict__ mats, unsigned long long* status, GjPass pass) {
  gj_la2_body<N, NWT, NPW, GjGlobalSrc<N>, NOPIV, GA>(nmat, mats, status, GjGlobalSrc<N>{mats}, pass);
}

// K4 face blocks assembled in place (assembly.py:994-1026): the face block
// sum_sides area_side * sum_q fw fphi_i fphi_j hh_q is built in the
// Gauss-Jordan CTA's working matrix (same DMMA contraction and the same
// accumulation order as k_precond_factor<.., INV = false>), so the block
// never round-trips through HBM before its inversion.  Also counts the
// non-symmetric blocks (the reference's Cholesky / LU choice statistic).
template <int P, int NT>
struct FaceBlockSrc {
  using D = Dims<P>;
  static constexpr int NB = D::NB, NQF = D::NQF, NFN = D::NFN;
  static constexpr int WMT = (NFN * NFN + 7) / 8, WKS = (NQF + 3) / 4, WNT = 4;
  // persistent tables in the extra shared memory; per-face staging in the
  // (then idle) U panel buffers
  static constexpr size_t extra_bytes = (size_t)(NQF * NFN + NQF + 2 * (NT / 32) + 2 + NFN) * 8;
  static constexpr int tmp_doubles = 2 * NQF * 25;
  Geo g;
  const double* hh;
  const double* hh_rem;
  const int* tidx_rem;
  const double* area_rem;
  int* n_unsym;
  __device__ __forceinline__ void init(double* ex, int tid, int nt) const {
    double* sFP = ex;
    double* sFw = sFP + NQF * NFN;
    for (int i = tid; i < NQF * NFN; i += nt) sFP[i] = g.fphi[i];
    for (int i = tid; i < NQF; i += nt) sFw[i] = g.fw[i];
  }
  // the next face's hh rows (both sides) towards L2
  __device__ __forceinline__ void prefetch(int f, int tid, int nt) const {
    constexpr int LN = (NQF * 25 * 8 + 127) / 128;
    for (int i = tid; i < 2 * LN; i += nt) {
      const int st = g.fsides[f * 2 + i / LN];
      if (st >= 0) prefetch_l2(reinterpret_cast<const char*>(hh + (size_t)st * NQF * 25) + (i % LN) * 128);
    }
  }
  __device__ __forceinline__ void load(int f, double* A, int S, double* ex, double* tmp, int tid, int nt) const {
    const double* sFP = ex;
    const double* sFw = sFP + NQF * NFN;
    double* sHH = tmp;                                // 2 sides x NQF x 25
    double* sRed = const_cast<double*>(sFw) + NQF;    // 2 * warps
    double* sArea = sRed + 2 * (NT / 32);
    int* sT = reinterpret_cast<int*>(sArea + 2);
    const int lane = tid & 31, warp = tid >> 5;
    // both sides staged at once
    for (int side = 0; side < 2; ++side) {
      const int st = g.fsides[f * 2 + side];
      double* hs = sHH + side * NQF * 25;
      int* ts = sT + side * NFN;
      if (st >= 0) {
        const int e = st / 4, k = st % 4;
        for (int i = tid; i < NQF * 25; i += nt) hs[(i % NQF) * 25 + i / NQF] = hh[((size_t)st * NQF) * 25 + i];
        for (int i = tid; i < NFN; i += nt) ts[i] = g.tidx[((size_t)e * 4 + k) * NFN + i];
        if (tid == 0) sArea[side] = g.area[(size_t)e * 4 + k];
      } else if (st != -1) {   // remote side of a halo face (partitioned runs)
        const int r = -2 - st;
        for (int i = tid; i < NQF * 25; i += nt) hs[(i % NQF) * 25 + i / NQF] = hh_rem[(size_t)r * NQF * 25 + i];
        for (int i = tid; i < NFN; i += nt) ts[i] = tidx_rem[(size_t)r * NFN + i];
        if (tid == 0) sArea[side] = area_rem[r];
      }
    }
    __syncthreads();
    // the sides one after the other, a warp per M tile: every entry of the
    // block receives exactly one term per side (tidx is a bijection per
    // side), so the first present side stores and the second adds: the
    // block is (term0) + term1, bit-identical to the former shared-memory
    // atomics onto zero (whose two orders give the same IEEE sum) without
    // their serialisation, and no zero fill is needed (padding rows and
    // columns of A stay zero from the kernel start)
    const bool has0 = g.fsides[f * 2] != -1;
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
      if (g.fsides[f * 2 + side] == -1) continue;
      const bool first = side == 0 || !has0;
      const double* hs = sHH + side * NQF * 25;
      const int* ts = sT + side * NFN;
      const double area = sArea[side];
      for (int mt = warp; mt < WMT; mt += NT / 32) {
        const int ija = mt * 8 + (lane >> 2);
        const bool rowok = ija < NFN * NFN;
        const int ia = rowok ? ija / NFN : 0, ja = rowok ? ija % NFN : 0;
        double c[WNT][2];
#pragma unroll
        for (int ntl = 0; ntl < WNT; ++ntl) c[ntl][0] = c[ntl][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < WKS; ++ks) {
          const int qa = ks * 4 + (lane & 3);
          const double a = (rowok && qa < NQF) ? (sFw[qa] * sFP[qa * NFN + ia]) * sFP[qa * NFN + ja] : 0.0;
#pragma unroll
          for (int ntl = 0; ntl < WNT; ++ntl) {
            const int n = ntl * 8 + (lane >> 2);
            const double b = (qa < NQF && n < 25) ? hs[qa * 25 + n] : 0.0;
            dmma_8x8x4(c[ntl], a, b);
          }
        }
        if (rowok) {
          const int rb = ts[ia] * 5, cb = ts[ja] * 5;
#pragma unroll
          for (int ntl = 0; ntl < WNT; ++ntl)
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int st2 = ntl * 8 + (lane & 3) * 2 + h2;
              if (st2 < 25) {
                double* dst = &A[(rb + st2 / 5) * S + cb + st2 % 5];
                const double v = area * c[ntl][h2];
                *dst = first ? v : *dst + v;
              }
            }
        }
      }
      __syncthreads();
    }
    __syncthreads();
    double amax = 0.0, dmax = 0.0;
    for (int idx = tid; idx < NB * NB; idx += nt) amax = fmax(amax, fabs(A[(idx / NB) * S + idx % NB]));
    // |a_rc - a_cr| along the diagonals c - r = d: the lanes of a warp walk
    // one diagonal, so both reads stride S + 1 (no bank conflicts)
    for (int d = 1 + warp; d < NB; d += NT / 32)
      for (int r = lane; r < NB - d; r += 32) dmax = fmax(dmax, fabs(A[r * S + r + d] - A[(r + d) * S + r]));
    for (int off = 16; off > 0; off >>= 1) {
      amax = fmax(amax, __shfl_down_sync(0xffffffffu, amax, off));
      dmax = fmax(dmax, __shfl_down_sync(0xffffffffu, dmax, off));
    }
    if (lane == 0) {
      sRed[warp] = amax;
      sRed[NT / 32 + warp] = dmax;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < NT / 32; ++w) {
        amax = fmax(amax, sRed[w]);
        dmax = fmax(dmax, sRed[NT / 32 + w]);
      }
      if (n_unsym && !(dmax <= 1e-12 * fmax(1.0, amax))) atomicAdd(n_unsym, 1);
    }
  }
};

template <int P, int NWT, int NPW, bool NOPIV = false>
__global__ void __launch_bounds__(32 * NWT, (Dims<P>::NB < 64 ? MHDG_GJ_MINB_SMALL : 2))
k_precond_gj(Geo g, int n_faces, const double* __restrict__ hh, const double* __restrict__ hh_rem,
             const int* __restrict__ tidx_rem, const double* __restrict__ area_rem, double* __restrict__ pinv,
             unsigned long long* status, int* n_unsym, GjPass pass) {
  static_assert(FaceBlockSrc<P, 32 * NWT>::tmp_doubles <= 2 * GJLA2<Dims<P>::NB, NWT, NPW>::UF, "staging");
  gj_la2_body<Dims<P>::NB, NWT, NPW, FaceBlockSrc<P, 32 * NWT>, NOPIV>(
      n_faces, pinv, status, FaceBlockSrc<P, 32 * NWT>{g, hh, hh_rem, tidx_rem, area_rem, n_unsym}, pass);
}

}  // namespace mhdg
