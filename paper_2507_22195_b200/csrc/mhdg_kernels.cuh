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
#include "mhdg_visc_math.cuh"

// Programmatic dependent launch on the condensed-matvec chain (k_face2<0> ->
// k_local_solve -> k_face2<1>) and the face-block preconditioner: each
// kernel launches while its producer drains, stages what does not depend on
// it (basis tables, face metadata), then blocks in pdl_wait() until the
// producer grid has completed and flushed.  Producers release at exit:
// measured at config 2, matvec 0.519 -> 0.512 ms; an explicit
// griddepcontrol.launch_dependents at each CTA's last batch was slower
// (0.521 ms: the early dependents hold SM slots), an L2 prefetch of the first
// S^-1 columns before the wait was neutral.  Without the launch attribute the
// wait is a no-op.
// INVARIANT at every pdl_wait() call site (tests/test_gpu_pdl.py builds the
// library with -DMHDG_PDL=0 and checks bit-identical operator outputs):
// before the wait a kernel may only READ immutable context tables (basis /
// facet tables, face ids, trace permutations, areas, rows, node-face maps)
// and WRITE its own shared memory / registers; every CTA executes the wait
// before touching any buffer a predecessor writes (x, z, gbuf, S^-1 inputs,
// r_w, r_q, y, hh, hw, hhat) and no CTA exits before it.
#ifndef MHDG_PDL
#define MHDG_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if MHDG_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

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
  const double* phit;  // (NN, NQ): phi transposed (coalesced per-point interpolation)
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
  const double* geo26; // (E, 50): det, J^-1 (9), normals (12), areas (4), tangent frames t1, t2 of the normals (24)
  const int* meta;     // (E, 8 + 4 NFN): face ids (4), trace permutations (4 NFN), boundary flags (4)
  int e_base;          // global index of macro 0 of this (sub-range) view, for error reports
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

// 8-byte asynchronous global -> shared copy (LDGSTS) and its completion wait
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(int* dst, const int* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

#ifdef MHDG_RES_TIMING
// phase clocks of the residual (experiment builds only): per group leader
__device__ unsigned long long g_res_clk[32];
#define RES_T(k)                                                   \
  do {                                                             \
    const long long t_ = clock64();                                \
    if (gtid == 0) atomicAdd(&g_res_clk[k], (unsigned long long)(t_ - t_prev)); \
    t_prev = t_;                                                   \
  } while (0)
#else
#define RES_T(k) \
  do {           \
  } while (0)
#endif

// pure (non-volatile) DMMA: lets the scheduler hoist the operand loads
__device__ __forceinline__ void dmma_8x8x4_nv(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// named barrier over one thread group (id 0 is __syncthreads)
__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Residual launch geometry.  A CTA holds NG independent groups of NW warps;
// each group processes EB macros per iteration and synchronises with its own
// named barrier, so the groups drift in phase against each other like
// separate CTAs would, while the basis tables (B in DMMA-fragment layout,
// phi^T for the per-point interpolation) are staged ONCE per CTA in shared
// memory instead of being re-read through a small L1 (with 4 CTAs x 51 KB of
// shared memory per SM the 51 KB of tables missed L1 a third of the time:
// 590 MB of L2 reads per launch at config 2 for 132 MB of DRAM traffic).
template <int P>
struct ResCfg {
  using D = Dims<P>;
  // macros per group iteration: enough quadrature points for the group's
  // threads at low degree (P = 1: 8 volume + 16 face points per macro)
  // (P = 4: two macros per 8-warp group: one macro's 100 face / 125 volume
  // points left half of the group's 256 threads waiting at the phase barrier,
  // 26% of the stall samples)
#ifndef MHDG_RES_EB1
#define MHDG_RES_EB1 16   // k = 1 macros per group iteration (A/B builds: 8)
#endif
  static constexpr int EB = (P >= 4) ? 2 : (P == 1 ? MHDG_RES_EB1 : (P == 2 ? 3 : 2));
  static constexpr int NW = (P >= 4) ? 8 : 4;      // warps per group
  static constexpr int GT = NW * 32;               // threads per group
  static constexpr int NG = (P >= 4) ? 2 : 4;      // groups per CTA
  static constexpr bool SB = P <= 3;               // basis tables in shared memory
  static constexpr int NT = NG * GT;
  static constexpr int MINB = 1;                   // resident CTAs per SM (register cap: 128 x 512 threads)
  // warps per macro in the contraction.  P = 2 has EB = 3 macros for 4 warps:
  // one job per macro left a warp idle (barrier stalls 19% of the samples), so
  // each macro is split four ways (K quarters of the volume test, one face each)
  static constexpr int WPM = (P == 2) ? 4 : (NW / EB > 0 ? NW / EB : 1);
  // P = 1: the tiles are too small for the tensor cores (NN = 4 of 8 columns,
  // one DMMA per face followed by a scattered epilogue: the contraction was
  // 42% of the kernel); one thread per output entry on the FP64 pipe instead
  static constexpr bool POINTWISE_TEST = (P == 1);
  static constexpr int NTILE = (D::NN + 7) / 8;    // DMMA N tiles over nodes (volume test)
  static constexpr int FMT = (2 * D::NFN + 7) / 8; // face test: M tiles over phi_face + fphi rows
  static constexpr int FKS = (D::NQF + 3) / 4;     // face test: K steps over face points
  static constexpr int AF_ = 4 * FMT * FKS * 32;   // face-test A fragments, lane-swizzled
  // B row stride: >= NN and = 4 (mod 16) so that the B-fragment reads
  // (lane = 4 n + kk -> word kk*RS + n) are free of bank conflicts
  static constexpr int RS = D::NN + ((4 - D::NN) % 16 + 16) % 16;
  static constexpr int GS = 21;                    // G row stride (odd)
  static constexpr int W_ = D::NN * 5, TR_ = 4 * D::NFN * 5, G_ = D::NQ * GS, H_ = 4 * D::NQF * 5,
                       FR_ = 4 * D::NFN * 5, VOL_ = WPM * D::NN * 5, GEO_ = 50;
  // w / trace (phase 1) and the face / volume partial rows (phases 2-3)
  // share one region; the far-field flux rows HG exist only with a
  // free-stream boundary (has_uinf)
  // w / trace / geometry of a batch arrive by cp.async in a staging region of
  // their own (STG_ per macro), read in place by phase 1; the face / volume
  // partial rows (phases 2-3) have theirs
  static constexpr int AREG = POINTWISE_TEST ? 0 : FR_ + VOL_;   // partial rows of the DMMA tests
  static constexpr int STG_ = W_ + TR_ + GEO_;
  static constexpr int per_macro_base = AREG + G_ + H_ + STG_;
  static constexpr int tables = 4 * D::NQF * D::FS + D::NQF * D::FS + D::NQ + D::NQF + AF_ +
                                (SB ? D::NQ * 4 * RS + D::NN * D::NQ : 0);
  static constexpr int per_macro_int = 4 + 4 * D::NFN + 4;   // x 2 slots (double-buffered)
  static constexpr int META = 4 + 4 * D::NFN + 4;
  static constexpr int table_int = 4 * D::NFN + 3 * D::NN;
  __host__ __device__ static constexpr int per_macro(int has_uinf) { return per_macro_base + (has_uinf ? H_ : 0); }
  // ng: groups of the launch (NG, fewer when the far-field rows of a
  // free-stream boundary would not fit: k = 3 with has_uinf runs 3 groups)
  __host__ __device__ static constexpr size_t bytes(int has_uinf, int ng = NG) {
    return (size_t)(tables + ng * EB * per_macro(has_uinf)) * 8 +
           (size_t)(table_int + ng * 2 * EB * per_macro_int) * 4;
  }
};

template <int P, int FK = -1>   // FK: flux kind fixed at compile time (-1: g.kind at run time)
__global__ void __launch_bounds__(ResCfg<P>::NT, ResCfg<P>::MINB)
k_residual(Geo g, const double* __restrict__ w, const double* __restrict__ trace,
           int has_stage, double alpha, const double* __restrict__ offset, int check,
           double* __restrict__ r_w, double* __restrict__ r_tr, unsigned long long* status) {
  using D = Dims<P>;
  using R = ResCfg<P>;
  constexpr int GT = R::GT, EB = R::EB, NN = D::NN, NQ = D::NQ, NFN = D::NFN, NQF = D::NQF;
  const int NT = blockDim.x, NG = NT / GT;   // groups of this launch (<= R::NG)
  constexpr int GS = R::GS, RS = R::RS;
  extern __shared__ __align__(16) double smem[];
  const int PM = R::per_macro(g.has_uinf);
  double* sPF = smem;                              // 4*NQF*FS
  double* sFP = sPF + 4 * NQF * D::FS;             // NQF*FS
  double* sQW = sFP + NQF * D::FS;                 // NQ
  double* sFW = sQW + NQ;                          // NQF
  double* sAF = sFW + NQF;                         // AF_
  double* sB = sAF + R::AF_;                       // NQ*4*RS (SB)
  double* sPT = sB + (R::SB ? NQ * 4 * RS : 0);    // NN*NQ   (SB)
  double* mball = smem + R::tables;                // NG * EB * PM
  int* sRows = (int*)(mball + NG * EB * PM);       // 4*NFN
  int* sNF = sRows + 4 * NFN;                      // 3*NN
  int* iball = sNF + 3 * NN;                       // NG * 2 * EB * per_macro_int
  const int tid = threadIdx.x, lane = tid & 31;
  // Optional: group g = the warps with warp id % NG == g: a warp issues on scheduler
  // warp id % 4, so with four groups each group owns one scheduler and its
  // warps move through the pointwise and the DMMA phases together (a
  // dependent DFMA chain sharing a scheduler with another group's DMMA
  // stream runs 5x slower: 8.8 -> 47.5 cycles per operation, measured).
  // Measured at n = 32 (session 5, ms, contiguous groups vs one group per
  // scheduler): ES k = 2 1.083 / 1.030, ES k = 3 1.996 / 1.940, KEPES k = 3
  // 2.194 / 2.231, ES k = 1 0.385 / 0.646: on for the ES instantiation at
  // k = 2, 3 (MHDG_RES_SCHED_GROUPS = 0 / 1 forces it off / on everywhere).
#ifdef MHDG_RES_SCHED_GROUPS
  constexpr bool SCHED = MHDG_RES_SCHED_GROUPS != 0;
#else
  constexpr bool SCHED = FK == FLUX_ES && (P == 2 || P == 3);
#endif
  const bool sched = SCHED && NG == 4;
  const int grp = sched ? (tid >> 5) % NG : tid / GT;
  const int gwarp = sched ? (tid >> 5) / NG : (tid % GT) >> 5;
  const int gtid = gwarp * 32 + lane;
  for (int i = tid; i < 4 * NQF * NFN; i += NT) sPF[(i / NFN) * D::FS + i % NFN] = g.pf[i];
  for (int i = tid; i < NQF * NFN; i += NT) sFP[(i / NFN) * D::FS + i % NFN] = g.fphi[i];
  for (int i = tid; i < NQ; i += NT) sQW[i] = g.qw[i];
  for (int i = tid; i < NQF; i += NT) sFW[i] = g.fw[i];
  for (int i = tid; i < 4 * NFN; i += NT) sRows[i] = g.rows[i];
  for (int i = tid; i < 3 * NN; i += NT) sNF[i] = g.nodef[i];
  // face-test A fragments: [k][mt][ks][lane], lane = 4 r + c holds
  // A[row = 8 mt + r][q = 4 ks + c] (row < NFN: phi_face[k][q][row],
  // row < 2 NFN: fphi[q][row - NFN], zero padding elsewhere)
  for (int i = tid; i < R::AF_; i += NT) {
    const int ln = i % 32, ks = (i / 32) % R::FKS, mt = (i / (32 * R::FKS)) % R::FMT, k = i / (32 * R::FKS * R::FMT);
    const int row = mt * 8 + (ln >> 2), q = ks * 4 + (ln & 3);
    double v = 0.0;
    if (q < NQF) {
      if (row < NFN) v = g.pf[(k * NQF + q) * NFN + row];
      else if (row < 2 * NFN) v = g.fphi[q * NFN + row - NFN];
    }
    sAF[i] = v;
  }
  if constexpr (R::SB) {
    for (int i = tid; i < NQ * 4 * NN; i += NT) sB[(i / NN) * RS + i % NN] = g.B[i];
    for (int i = tid; i < NN * NQ; i += NT) sPT[i] = g.phit[i];
  }
  __syncthreads();
  const double gam = g.gamma;
  const double* __restrict__ Bt = R::SB ? sB : g.B;
  const int bstride = R::SB ? RS : NN;
  double* mb = mball + grp * EB * PM;
  int* ib = iball + grp * 2 * EB * R::per_macro_int;
  const int bar_id = 1 + grp;
  auto gsync = [&]() { group_sync(bar_id, GT); };

  auto FR = [&](int m) { return mb + m * PM; };          // face partial rows (phases 2-3)
  auto VOL = [&](int m) { return FR(m) + R::FR_; };
  auto G = [&](int m) { return FR(m) + R::AREG; };
  auto H = [&](int m) { return G(m) + R::G_; };
  auto W = [&](int m) { return H(m) + R::H_; };          // staging: w, trace, geometry (cp.async)
  auto TR = [&](int m) { return W(m) + R::W_; };
  auto GEO = [&](int m) { return TR(m) + R::TR_; };
  auto HG = [&](int m) { return GEO(m) + R::GEO_; };     // only with has_uinf
  // meta (face ids, trace permutations, boundary flags) is double-buffered:
  // slot `cur` serves the batch being computed, slot `cur ^ 1` receives the
  // next batch's, whose w / trace / geometry are prefetched into registers
  // during the contraction phase (no dependent global round trip left on
  // the critical path except the first batch's).
  int cur = 0;
  auto FID = [&](int m) { return ib + (cur * EB + m) * R::per_macro_int; };
  auto TID = [&](int m) { return FID(m) + 4; };
  auto BND = [&](int m) { return TID(m) + 4 * NFN; };
  auto meta_ld = [&](int e0n, int i, int& v) {     // i over EB*META (packed per-macro meta)
    if (e0n + i / R::META < g.E) v = g.meta[(size_t)e0n * R::META + i];
  };
  // The next batch's w / geometry / trace values go straight from global to
  // the staging region with cp.async (no registers: as register prefetches
  // they were spilled at the 128-register cap, and the spill store waited for
  // each load, 14% of the kernel's stall samples).  Issued after the barrier
  // that ends phase 1 (the staging region is read only by phase 1), waited
  // for at the top of the next batch.
  auto prefetch_wg = [&](int e0n) {                 // w and geometry
    const int nmn = min(EB, g.E - e0n);
    for (int i = gtid; i < nmn * (NN * 5 / 1); i += GT)
      cp_async8(W(i / (NN * 5)) + i % (NN * 5), w + (size_t)e0n * NN * 5 + i);
    for (int i = gtid; i < nmn * R::GEO_; i += GT)
      cp_async8(GEO(i / R::GEO_) + i % R::GEO_, g.geo26 + (size_t)e0n * R::GEO_ + i);
  };
  auto prefetch_tr = [&](int e0n, int slot) {       // trace values through slot's meta
    const int nmn = min(EB, g.E - e0n);
    for (int i = gtid; i < nmn * 4 * NFN * 5; i += GT) {
      const int m = i / (4 * NFN * 5), r = i % (4 * NFN * 5);
      const int k = r / (NFN * 5), j = (r / 5) % NFN, s = r % 5;
      const int* mt = ib + (slot * EB + m) * R::per_macro_int;
      cp_async8(TR(m) + r, trace + ((size_t)mt[k] * NFN + mt[4 + k * NFN + j]) * 5 + s);
    }
  };
  const int gidx = blockIdx.x * NG + grp, gstride = gridDim.x * NG;
  {   // first batch: meta, then its data
    const int e00 = gidx * EB;
    if (e00 < g.E) {
      for (int i = gtid; i < EB * R::META; i += GT) {
        int v = 0;
        meta_ld(e00, i, v);
        ib[(i / R::META) * R::per_macro_int + i % R::META] = v;
      }
      gsync();
      prefetch_wg(e00);
      prefetch_tr(e00, 0);
    }
  }

#ifdef MHDG_RES_TIMING
  long long t_prev = clock64();
#endif
  for (int e0 = gidx * EB; e0 < g.E; e0 += gstride * EB) {
    const int nm = min(EB, g.E - e0);
    const int e1 = e0 + gstride * EB;
    cp_async_wait_all();
    gsync();
    RES_T(0);
    // next batch's meta into the other slot (free since the barrier above),
    // asynchronously under phase 1
    if (e1 < g.E) {
      const int nmn = min(EB, g.E - e1);
      for (int i = gtid; i < nmn * R::META; i += GT)
        cp_async4(ib + ((cur ^ 1) * EB + i / R::META) * R::per_macro_int + i % R::META,
                  g.meta + (size_t)e1 * R::META + i);
    }
    RES_T(1);

    // ---- 1a. face quadrature points: two-point flux, weighted
    for (int it = gtid; it < nm * 4 * NQF; it += GT) {
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
      if (!to_conservative(wq, g.form, gam, u)) report(status, 1 + k, 0, e + g.e_base);
      if (!to_conservative(whq, g.form, gam, uh)) report(status, 1 + k, 1, e + g.e_base);
      if (check && !admissible(u, gam)) report(status, 1 + k, 2, e + g.e_base);
      if (check && !admissible(uh, gam)) report(status, 1 + k, 3, e + g.e_base);
      const double* geo = GEO(m);
      const double n[3] = {geo[10 + k * 3], geo[11 + k * 3], geo[12 + k * 3]};
      double fh[5];
      numerical_flux(FK >= 0 ? FK : g.kind, u, uh, n, gam, fh, g.form == FORM_ENTROPY ? wq : nullptr,
                     g.form == FORM_ENTROPY ? whq : nullptr, geo + 26 + 6 * k);
      const double fwq = sFW[q] * geo[22 + k];
      double* h = H(m) + kq * 5;
#pragma unroll
      for (int s = 0; s < 5; ++s) h[s] = fwq * fh[s];
      if (g.has_uinf && BND(m)[k]) {
        const double mn[3] = {-n[0], -n[1], -n[2]};
        double gh[5];
        numerical_flux(FK >= 0 ? FK : g.kind, g.uinf, uh, mn, gam, gh);
#pragma unroll
        for (int s = 0; s < 5; ++s) HG(m)[kq * 5 + s] = fwq * gh[s];
      }
    }
    RES_T(2);
    // ---- 1b. volume quadrature points: reference-space flux + temporal term
    for (int it = gtid; it < nm * NQ; it += GT) {
      const int m = it / NQ, q = it % NQ, e = e0 + m;
      const double* sw = W(m);
      // the stage offset of this point first: its global-load latency runs
      // under the interpolation and the flux evaluation
      double off[5] = {0, 0, 0, 0, 0};
      if (has_stage && offset) {
#pragma unroll
        for (int s = 0; s < 5; ++s) off[s] = __ldcs(offset + ((size_t)e * NQ + q) * 5 + s);
      }
      double wq[5] = {0, 0, 0, 0, 0};
#pragma unroll 4
      for (int i = 0; i < NN; ++i) {
        const double a = R::SB ? sPT[i * NQ + q] : __ldg(g.phit + (size_t)i * NQ + q);
#pragma unroll
        for (int s = 0; s < 5; ++s) wq[s] += a * sw[i * 5 + s];
      }
      double u[5];
      if (!to_conservative(wq, g.form, gam, u)) report(status, 0, 0, e + g.e_base);
      if (check && !admissible(u, gam)) report(status, 0, 2, e + g.e_base);
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
          if (offset) tmp = tmp + off[s];
          tmp = vw * tmp;
        }
        gr[15 + s] = tmp;
      }
    }
    // the next batch's meta (issued at the top of this batch) has landed
    cp_async_wait_all();
    RES_T(3);
    gsync();
    RES_T(4);
    if (e1 < g.E) {   // phase 1 is over for the whole group: the staging region is free
      prefetch_wg(e1);
      prefetch_tr(e1, cur ^ 1);
      if (has_stage && offset) {   // the next batch's stage offsets towards L2
        const int nmn = min(EB, g.E - e1);
        for (int i = gtid * 16; i < nmn * NQ * 5; i += GT * 16) prefetch_l2(offset + (size_t)e1 * NQ * 5 + i);
      }
    }

    if constexpr (R::POINTWISE_TEST) {
      // ---- 2'. tests on the FP64 pipe, one thread per output entry:
      // r_w[m][i][s] = sum_(q,kk) G[q][kk][s] B[q][kk][i] + the face rows of
      // the faces that contain node i; r_trace side contributions per (k, j, s)
      for (int o = gtid; o < nm * NN * 5; o += GT) {
        const int m = o / (NN * 5), is = o % (NN * 5), i = is / 5, s = is % 5;
        const double* gm = G(m) + s;
        const double* bcol = Bt + i;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          a0 = fma(gm[q * GS], bcol[(q * 4) * bstride], a0);
          a1 = fma(gm[q * GS + 5], bcol[(q * 4 + 1) * bstride], a1);
          a0 = fma(gm[q * GS + 10], bcol[(q * 4 + 2) * bstride], a0);
          a1 = fma(gm[q * GS + 15], bcol[(q * 4 + 3) * bstride], a1);
        }
        const double* hm = H(m) + s;
        double f0 = 0.0;
#pragma unroll
        for (int c2 = 0; c2 < 3; ++c2) {
          const int kj = sNF[i * 3 + c2];
          if (kj < 0) break;
          const int k = kj / NFN, j = kj % NFN;
          double f1 = 0.0;
#pragma unroll
          for (int q = 0; q < NQF; ++q) f1 = fma(sPF[(k * NQF + q) * D::FS + j], hm[(k * NQF + q) * 5], f1);
          f0 += f1;
        }
        r_w[(size_t)e0 * NN * 5 + o] = (a0 + a1) + f0;
      }
      for (int o = gtid; o < nm * 4 * NFN * 5; o += GT) {
        const int m = o / (4 * NFN * 5), r = o % (4 * NFN * 5);
        const int k = r / (NFN * 5), j = (r / 5) % NFN, s = r % 5;
        const double* hk = H(m) + k * NQF * 5 + s;
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < NQF; ++q) v = fma(sFP[q * D::FS + j], hk[q * 5], v);
        if (g.has_uinf && BND(m)[k]) {
          const double* gk = HG(m) + k * NQF * 5 + s;
          double vg = 0.0;
#pragma unroll
          for (int q = 0; q < NQF; ++q) vg = fma(sFP[q * D::FS + j], gk[q * 5], vg);
          v += vg;
        }
        atomicAdd(&r_tr[((size_t)FID(m)[k] * NFN + TID(m)[k * NFN + j]) * 5 + s], v);
      }
      RES_T(5);
    } else {
    // ---- 2. contraction on the FP64 tensor cores, all WPM warps of a macro
    // alike: warp r takes the volume-test K range q in [r NQ/WPM, (r+1)
    // NQ/WPM) and the face tests of faces k = r, r + WPM, ...
    for (int job = gwarp; job < nm * R::WPM; job += R::NW) {
      const int m = job / R::WPM, role = job % R::WPM;
      {
        {   // volume test: C[s][i] += sum_k G^T[s][k] B[k][i], k = (q, kk)
          const int q0 = role * NQ / R::WPM, q1 = (role + 1) * NQ / R::WPM;
          const int s_a = lane >> 2, kk = lane & 3;
          double c[R::NTILE][2];
#pragma unroll
          for (int t = 0; t < R::NTILE; ++t) c[t][0] = c[t][1] = 0.0;
          const double* gm = G(m);
          for (int q = q0; q < q1; ++q) {
            const double a = s_a < 5 ? gm[q * GS + kk * 5 + s_a] : 0.0;
            const double* brow = Bt + ((size_t)q * 4 + kk) * bstride;
#pragma unroll
            for (int t = 0; t < R::NTILE; ++t) {
              const int i = t * 8 + (lane >> 2);
              const double b = i < NN ? (R::SB ? brow[i] : __ldg(brow + i)) : 0.0;
              dmma_8x8x4_nv(c[t], a, b);
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
        }
        // face tests, per face k: C[row][s] = sum_q A[row][q] H[k][q][s] with
        // rows 0..NFN-1 = phi_face (the r_w face rows) and NFN..2NFN-1 = fphi
        // (this side's r_trace contribution); A fragments come pre-swizzled
        // from sAF, the far-field rows HG (free-stream faces only) take a
        // second pass over the fphi rows
        const double* hm = H(m);
        const int* fid = FID(m);
        const int* tdx = TID(m);
        const int kq_ = lane & 3, n_ = lane >> 2;
        for (int k = role; k < 4; k += R::WPM) {
          const bool bnd = g.has_uinf && BND(m)[k];
          double c[R::FMT][2], cg[R::FMT][2];
#pragma unroll
          for (int t = 0; t < R::FMT; ++t) c[t][0] = c[t][1] = cg[t][0] = cg[t][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < R::FKS; ++ks) {
            const int q = ks * 4 + kq_;
            const double hb = (n_ < 5 && q < NQF) ? hm[(k * NQF + q) * 5 + n_] : 0.0;
#pragma unroll
            for (int t = 0; t < R::FMT; ++t)
              dmma_8x8x4_nv(c[t], sAF[((k * R::FMT + t) * R::FKS + ks) * 32 + lane], hb);
          }
          if (bnd) {
#pragma unroll
            for (int ks = 0; ks < R::FKS; ++ks) {
              const int q = ks * 4 + kq_;
              const double hb = (n_ < 5 && q < NQF) ? HG(m)[(k * NQF + q) * 5 + n_] : 0.0;
#pragma unroll
              for (int t = 0; t < R::FMT; ++t)
                dmma_8x8x4_nv(cg[t], sAF[((k * R::FMT + t) * R::FKS + ks) * 32 + lane], hb);
            }
          }
#pragma unroll
          for (int t = 0; t < R::FMT; ++t)
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int row = t * 8 + n_, sc = kq_ * 2 + h2;
              if (sc < 5) {
                if (row < NFN) {
                  FR(m)[(k * NFN + row) * 5 + sc] = c[t][h2];
                } else if (row < 2 * NFN) {
                  const int j = row - NFN;
                  const double v = bnd ? c[t][h2] + cg[t][h2] : c[t][h2];
                  atomicAdd(&r_tr[((size_t)fid[k] * NFN + tdx[k * NFN + j]) * 5 + sc], v);
                }
              }
            }
        }
      }
    }
#ifdef MHDG_RES_TIMING
    if (gtid == 32) atomicAdd(&g_res_clk[8], (unsigned long long)(clock64() - t_prev));
#endif
    RES_T(5);
    gsync();
    RES_T(6);
    // ---- 3. r_w = volume part + face parts (tile order)
    for (int o = gtid; o < nm * NN * 5; o += GT) {
      const int m = o / (NN * 5), is = o % (NN * 5), i = is / 5, s = is % 5;
      double r = VOL(m)[is];
#pragma unroll
      for (int d2 = 1; d2 < R::WPM; ++d2) r += VOL(m)[d2 * NN * 5 + is];
#pragma unroll
      for (int c2 = 0; c2 < 3; ++c2) {
        const int kj = sNF[i * 3 + c2];
        if (kj < 0) break;
        r += FR(m)[kj * 5 + s];
      }
      r_w[(size_t)e0 * NN * 5 + o] = r;
    }
    RES_T(7);
    }   // DMMA tests
    cur ^= 1;
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
            unsigned long long* status, int do_gj = 1) {
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
        numerical_flux(g.kind, ud, uhd, n, gam, fd, g.form == FORM_ENTROPY ? wd : nullptr,
                       g.form == FORM_ENTROPY ? whd : nullptr);
        const size_t base = ((size_t)e * 4 + k) * 25 * D::NQF + q;   // ten layout (E,4,25,NQF)
        if (which == 0) {
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            hw_out[base + (s * 5 + t) * D::NQF] = fd[s].d;
            sHW[q * 25 + s * 5 + t] = fd[s].d;
          }
        } else {
          double hh[5];
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            hhat_out[base + (s * 5 + t) * D::NQF] = fd[s].d;
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
          for (int s = 0; s < 5; ++s) hh_out[base + (s * 5 + t) * D::NQF] = hh[s];
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

    if (!do_gj) {   // S row-major for a separate (blocked) inversion
      double* out = sinv + (size_t)e * NM * NM;
      for (int o = tid; o < NM * NM; o += NT) out[o] = S[o];
      continue;
    }
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
// Register-blocked Gauss-Jordan inverse with implicit partial pivoting.
// The N x N row-major matrix in shared memory A is distributed over a
// TR x TC thread grid (thread (tr, tc) owns rows tr + TR a, columns
// tc + TC b).  Step k: the pivot is the unused row with the largest |a_rk|
// (first on ties, LAPACK idamax semantics), found redundantly by every warp;
// no rows are swapped.  The result Y is written back to A with the pivot
// sequence q (q[k] = pivot row of step k); then A^-1[r][c] = Y[q[r]][q^-1[c]]
// (checked in numpy, tests/test_tables.py::test_implicit_pivot_gauss_jordan).
// Returns false if a pivot is zero / non-finite.
// ===========================================================================
template <int N, int TR, int TC>
struct GJDims {
  static constexpr int RA = (N + TR - 1) / TR, CB = (N + TC - 1) / TC;
  static constexpr int NPR = TR * RA, NPC = TC * CB;   // padded extents
  static constexpr int NI = (N + 31) / 32;
};

// w: this thread's register tile, loaded by the caller (padding = 0).
// colbuf: 2*NPR doubles, rowbuf: 2*NPC doubles (shared).  Writes q[N].
template <int N, int TR, int TC>
__device__ bool gj_inverse_reg(double (&w)[GJDims<N, TR, TC>::RA][GJDims<N, TR, TC>::CB], double* colbuf,
                               double* rowbuf, int* q, int* sflag) {
  using G = GJDims<N, TR, TC>;
  constexpr int RA = G::RA, CB = G::CB, NI = G::NI;
  const int tid = threadIdx.x, lane = tid & 31;
  const bool act = tid < TR * TC;
  const int tr = act ? tid / TC : 0, tc = act ? tid % TC : 0;
  for (int i = tid; i < 2 * G::NPR; i += blockDim.x) colbuf[i] = 0.0;
  for (int i = tid; i < 2 * G::NPC; i += blockDim.x) rowbuf[i] = 0.0;
  __syncthreads();
  unsigned used = 0u;
  bool ok = true;
  for (int k = 0; k < N; ++k) {
    const int cb = (k & 1) * G::NPR, rb = (k & 1) * G::NPC;
    // 1. owners of column k publish it and clear their copy (the new column
    //    k is -pinv * col for r != p and pinv on the pivot row)
    if (act && tc == k % TC) {
      const int kb = k / TC;
#pragma unroll
      for (int a = 0; a < RA; ++a) {
        double v = 0.0;
#pragma unroll
        for (int b2 = 0; b2 < CB; ++b2)
          if (b2 == kb) { v = w[a][b2]; w[a][b2] = 0.0; }
        colbuf[cb + tr + TR * a] = v;
      }
    }
    __syncthreads();
    // 2. pivot: unused row with the largest |a_rk|, first on ties (every warp)
    double best = -1.0;
    int bi = N;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int r = lane + 32 * i;
      if (r < N && !((used >> i) & 1u)) {
        const double v = fabs(colbuf[cb + r]);
        if (v > best) { best = v; bi = r; }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const int p = bi < N ? bi : 0;
    if ((p & 31) == lane) used |= 1u << (p >> 5);
    const double piv = colbuf[cb + p];
    if (!(fabs(piv) > 0.0) || !isfinite(piv)) ok = false;
    if (tid == 0) q[k] = p;
    // 3. pivot row owners scale the row and publish it
    if (act && tr == p % TR) {
      const int pa = p / TR;
      const double pinv = 1.0 / piv;
#pragma unroll
      for (int b2 = 0; b2 < CB; ++b2) {
        const int c = tc + TC * b2;
        double v = 0.0;
#pragma unroll
        for (int a = 0; a < RA; ++a)
          if (a == pa) v = w[a][b2];
        v = (c == k ? 1.0 : v) * pinv;
#pragma unroll
        for (int a = 0; a < RA; ++a)
          if (a == pa) w[a][b2] = v;
        rowbuf[rb + c] = v;
      }
    }
    __syncthreads();
    // 4. rank-1 update of every other row: pure FMAs
    if (act) {
      double rv[CB];
#pragma unroll
      for (int b2 = 0; b2 < CB; ++b2) rv[b2] = rowbuf[rb + tc + TC * b2];
#pragma unroll
      for (int a = 0; a < RA; ++a) {
        const int r = tr + TR * a;
        const double cr = (r == p) ? 0.0 : colbuf[cb + r];
#pragma unroll
        for (int b2 = 0; b2 < CB; ++b2) w[a][b2] -= rv[b2] * cr;
      }
    }
  }
  if (tid == 0) *sflag = ok ? 0 : 1;
  __syncthreads();
  return *sflag == 0;
}

// store A^-1 column-major from the implicit-pivot result Y in shared memory:
// out[c*N + r] = Y[q[r]][qinv[c]]; also reports non-finite entries
template <int N, int NT>
__device__ bool gj_store_colmajor(const double* Y, const int* q, int* qinv, double* out) {
  for (int k = threadIdx.x; k < N; k += NT) qinv[q[k]] = k;
  __syncthreads();
  int bad = 0;
  for (int o = threadIdx.x; o < N * N; o += NT) {
    const int c = o / N, r = o % N;
    const double v = Y[q[r] * N + qinv[c]];
    bad |= !isfinite(v);
    out[o] = v;
  }
  return __syncthreads_or(bad) == 0;
}

// ===========================================================================
// K2 v2 (P <= 3): linearization with the S assembly on the FP64 tensor cores.
//   pointwise : C[q][kk][st] (kk=0..2: -vol_w J^-1 dF/dw, kk=3: weight vol_w du/dw)
//               by forward-mode duals, st = s*5 + t
//   stage 1   : D[q][i][st] = sum_kk B[q][kk][i] C[q][kk][st]        (DMMA, K = 4)
//   stage 2   : S_st[i][j] += sum_q D[q][i][st] phi[q][j]            (DMMA, per q chunk)
//               accumulated in registers across chunks
//   faces     : hw/hhat/hh tensors + face blocks of S (as in v1)
//   inverse   : k_gj_blocked (mhdg_gj_blocked.cuh), implicit pivoting
// ===========================================================================
#ifndef MHDG_LIN2_PAD
#define MHDG_LIN2_PAD 1
#endif
// C row kk rotated by 4 kk columns: a half-warp's stage-1 B-fragment loads
// (four kk rows x four columns) then hit 16 distinct bank pairs
#define LIN2_CI(kk, col) ((kk) * CS + (L::ROT ? (((col) + 4 * (kk)) & 31) : (col)))
#ifndef MHDG_LIN2_PREFETCH
#define MHDG_LIN2_PREFETCH 0   // L2 prefetch of the next macro's inputs (measured: 115.0 vs 114.3 ms, off)
#endif
#ifndef MHDG_LIN2_FB_PAIR
#define MHDG_LIN2_FB_PAIR 1   // face-block units per warp pass (1 or 2: measured equal)
#endif
#ifndef MHDG_LIN2_NW
#define MHDG_LIN2_NW 8   // 10 warps (whole dual passes) measured slower: 168-register cap spills
#endif
// k = 4 (NM = 175): S (245 KB) does not fit shared memory; it is assembled
// in place in the S^-1 buffer (GS: L2-resident per CTA, the blocked
// Gauss-Jordan inverts it there), C rows are unpadded (CS = 25, the
// st >= 25 fragment lanes read 0) and the (st, i-tile) pairs run in two
// passes so that the stage-2 accumulators fit the register file.
template <int P>
struct Lin2 {
  using D = Dims<P>;
  static constexpr bool GS = (size_t)D::NM * D::NM * 8 > 100 * 1024;   // S in global memory
  static constexpr bool ROT = MHDG_LIN2_PAD && !GS;    // rotated C rows (needs CS = 32)
  static constexpr int NW = MHDG_LIN2_NW, NT = 32 * NW;
  static constexpr int NNP = (D::NN + 7) / 8 * 8;      // padded nodes
  static constexpr int IT = NNP / 8;                    // node tiles
  static constexpr int QC = 8;                          // q chunk (2 k-steps)
  static constexpr int NCH = (D::NQ + QC - 1) / QC;
  static constexpr int CS = GS ? 25 : 32;                // C row (st padded)
  // D row stride (doubles): NNP + 4, so the stage-1 stores of the four
  // (lane & 3) st columns and the stage-2 loads of the four q rows fall on
  // distinct bank pairs (NNP = 0 mod 8 put all four on one)
  static constexpr int DS = MHDG_LIN2_PAD ? NNP + 4 : NNP;
  static constexpr int NPAIR = 25 * IT;                  // (st, i-tile) pairs
  static constexpr int NPASS = GS ? 2 : 1;               // passes over the pairs
  static constexpr int PPW = ((NPAIR + NW - 1) / NW + NPASS - 1) / NPASS;   // pairs per warp and pass
  // shared memory (doubles)
  static constexpr int S_ = GS ? 0 : D::NM * D::NM;
  static constexpr int C_ = D::NQ * 4 * CS;
  static constexpr int DD_ = QC * 25 * DS;
  static constexpr int doubles = S_ + C_ + DD_ + D::NN * 5 + 4 * D::NFN * 5 + 4 * D::NQF * D::FS +
                                 D::NQF * D::FS + D::NQ + D::NQF + 4 * D::NQF * 25 +
                                 (GS ? 0 : 4 * D::NM) + 32;
  static constexpr int ints = 4 * D::NFN + 4 + 4 * D::NFN + 4 + 2 * D::NM + 4;
  static constexpr size_t bytes = (size_t)doubles * 8 + ints * 4 + 16 + D::NN * 15 * 8;
};

// One volume quadrature point and dual direction t (it = 5 q + t) of the
// linearization: the C rows  -vol_w J^-1 dF/dw_t  (kk = 0..2) and
// weight vol_w du/dw_t  (kk = 3) of point q, written into the macro's C block
// (shared memory in the fused kernel, the macro's S^-1 storage in the split
// pointwise kernel).  PADZ: also zero this item's share of the st >= 25
// padding columns (the split kernel fills a fresh block).
template <int P, bool VISC, bool PADZ>
__device__ __forceinline__ void lin2_volume_item(const Geo& g, const ViscGeo& vg, int it, const double* __restrict__ sW,
                                                 const double* __restrict__ sQn, const double* __restrict__ sQW,
                                                 const double* __restrict__ sGeo, double weight, double* sC) {
  using D = Dims<P>;
  using L = Lin2<P>;
  constexpr int NN = D::NN, CS = L::CS;
  const double* __restrict__ Bt = g.B;
  const double gam = g.gamma;
  const int q = it / 5, t = it % 5;
  const double* ph = Bt + ((size_t)q * 4 + 3) * NN;
  double wq[5] = {0, 0, 0, 0, 0};
  for (int i = 0; i < NN; ++i) {
    const double a = __ldg(ph + i);
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2) wq[s2] += a * sW[i * 5 + s2];
  }
  Dual wd[5], ud[5];
#pragma unroll
  for (int s2 = 0; s2 < 5; ++s2) wd[s2] = mk(wq[s2], s2 == t ? 1.0 : 0.0);
  to_conservative(wd, g.form, gam, ud);
  Dual F[5][3];
  flux(ud, gam, F);
  if (VISC) {
    double qq[5][3];
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2) qq[s2][0] = qq[s2][1] = qq[s2][2] = 0.0;
    for (int i = 0; i < NN; ++i) {
      const double a = __ldg(ph + i);
#pragma unroll
      for (int s2 = 0; s2 < 5; ++s2)
#pragma unroll
        for (int b = 0; b < 3; ++b) qq[s2][b] += a * sQn[i * 15 + s2 * 3 + b];
    }
    Dual Gv[5][3];
    visc_G(vg, g.form, wd, ud, qq, gam, Gv);
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2)
#pragma unroll
      for (int a = 0; a < 3; ++a) F[s2][a] = F[s2][a] + Gv[s2][a];
  }
  const double vw = sQW[q] * sGeo[0];
  double* C = sC + (size_t)q * 4 * CS;
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    const double j0 = sGeo[1 + kk * 3], j1 = sGeo[2 + kk * 3], j2 = sGeo[3 + kk * 3];
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2)
      C[LIN2_CI(kk, s2 * 5 + t)] = -(vw * ((j0 * F[s2][0].d + j1 * F[s2][1].d) + j2 * F[s2][2].d));
  }
#pragma unroll
  for (int s2 = 0; s2 < 5; ++s2) C[LIN2_CI(3, s2 * 5 + t)] = weight * (vw * ud[s2].d);
  if (PADZ && CS > 25) {
    for (int col = 25 + t; col < CS; col += 5)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) C[LIN2_CI(kk, col)] = 0.0;
  }
}

// One face quadrature point, dual direction t and side (it4 = ((k NQF + q) 2
// + which) 5 + t): the hw / hhat / hh tensor entries of tile k at point q
// (assembly.py:846-940); sHW (optional) stages the hw rows for the S face
// blocks of the fused kernel.
template <int P, bool VISC, int FK>
__device__ __forceinline__ void lin2_face_item(const Geo& g, const ViscGeo& vg, int e, int it4,
                                               const double* __restrict__ sW, const double* __restrict__ sTR,
                                               const double* __restrict__ sQn, const double* __restrict__ sPF,
                                               const double* __restrict__ sFP, const int* __restrict__ sRows,
                                               const double* __restrict__ sGeo, const int* __restrict__ sBnd,
                                               double ptc, double* __restrict__ hw_out,
                                               double* __restrict__ hhat_out, double* __restrict__ hh_out,
                                               double* sHW) {
  using D = Dims<P>;
  constexpr int NFN = D::NFN, NQF = D::NQF;
  const double gam = g.gamma;
  const int k = it4 / (NQF * 10), it = it4 % (NQF * 10);
  const double n[3] = {sGeo[10 + k * 3], sGeo[11 + k * 3], sGeo[12 + k * 3]};
  double* sHWk = sHW ? sHW + k * NQF * 25 : nullptr;
  const int q = it / 10, t = (it % 10) % 5, which = (it % 10) / 5;
  const double* pf = sPF + (k * NQF + q) * D::FS;
  const double* fp = sFP + q * D::FS;
  double wq[5] = {0, 0, 0, 0, 0}, whq[5] = {0, 0, 0, 0, 0};
  for (int j = 0; j < NFN; ++j) {
    const double a = pf[j], b = fp[j];
    const int row = sRows[k * NFN + j];
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2) {
      wq[s2] += a * sW[row * 5 + s2];
      whq[s2] += b * sTR[(k * NFN + j) * 5 + s2];
    }
  }
  Dual wd[5], whd[5], ud[5], uhd[5], fd[5];
#pragma unroll
  for (int s2 = 0; s2 < 5; ++s2) {
    wd[s2] = mk(wq[s2], (which == 0 && s2 == t) ? 1.0 : 0.0);
    whd[s2] = mk(whq[s2], (which == 1 && s2 == t) ? 1.0 : 0.0);
  }
  to_conservative(wd, g.form, gam, ud);
  to_conservative(whd, g.form, gam, uhd);
  numerical_flux(FK >= 0 ? FK : g.kind, ud, uhd, n, gam, fd, g.form == FORM_ENTROPY ? wd : nullptr,
                 g.form == FORM_ENTROPY ? whd : nullptr);
  if (VISC) {
    double qq[5][3];
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2) qq[s2][0] = qq[s2][1] = qq[s2][2] = 0.0;
    for (int j = 0; j < NFN; ++j) {
      const double a = pf[j];
      const int row = sRows[k * NFN + j];
#pragma unroll
      for (int s2 = 0; s2 < 5; ++s2)
#pragma unroll
        for (int b = 0; b < 3; ++b) qq[s2][b] += a * sQn[row * 15 + s2 * 3 + b];
    }
    Dual Gv[5][3];
    visc_G(vg, g.form, wd, ud, qq, gam, Gv);
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2) {
      const Dual gn = (Gv[s2][0] * n[0] + Gv[s2][1] * n[1]) + Gv[s2][2] * n[2];
      fd[s2] = fd[s2] + (gn - (0.5 * vg.pdiag[s2]) * (whd[s2] - wd[s2]));
    }
  }
  const size_t base = ((size_t)e * 4 + k) * 25 * NQF + q;   // ten layout (E,4,25,NQF)
  if (which == 0) {
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2) {
      hw_out[base + (s2 * 5 + t) * NQF] = fd[s2].d;
      if (sHWk) sHWk[q * 25 + s2 * 5 + t] = fd[s2].d;
    }
  } else {
    double hv[5];
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2) {
      hhat_out[base + (s2 * 5 + t) * NQF] = fd[s2].d;
      hv[s2] = fd[s2].d;
    }
    if (sBnd[k] && g.has_uinf) {
      Dual ui[5], gd[5];
#pragma unroll
      for (int s2 = 0; s2 < 5; ++s2) ui[s2] = mk(g.uinf[s2], 0.0);
      const double mn[3] = {-n[0], -n[1], -n[2]};
      numerical_flux(FK >= 0 ? FK : g.kind, ui, uhd, mn, gam, gd);
      if (VISC) {
        double winf[5];
        if (g.form == FORM_ENTROPY) entropy_vars(g.uinf, gam, winf);
        else for (int s2 = 0; s2 < 5; ++s2) winf[s2] = g.uinf[s2];
#pragma unroll
        for (int s2 = 0; s2 < 5; ++s2) gd[s2] = gd[s2] + (0.0 - (0.5 * vg.pdiag[s2]) * (whd[s2] - winf[s2]));
      }
#pragma unroll
      for (int s2 = 0; s2 < 5; ++s2) hv[s2] = hv[s2] + gd[s2].d;
    }
    if (ptc != 0.0) {
#pragma unroll
      for (int s2 = 0; s2 < 5; ++s2) hv[s2] = hv[s2] + (-ptc * uhd[s2].d);
    }
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2) hh_out[base + (s2 * 5 + t) * NQF] = hv[s2];
  }
}

template <int P, bool VISC, int FK = -1>   // FK: flux kind fixed at compile time (-1: run time)
__global__ void __launch_bounds__(32 * MHDG_LIN2_NW, 1)
k_linearize2(Geo g, ViscGeo vg, const double* __restrict__ w, const double* __restrict__ qn,
             const double* __restrict__ trace, double weight,
             double ptc, double* __restrict__ sinv, double* __restrict__ hw_out,
             double* __restrict__ hhat_out, double* __restrict__ hh_out, unsigned long long* status) {
  using D = Dims<P>;
  using L = Lin2<P>;
  constexpr int NN = D::NN, NQ = D::NQ, NM = D::NM, NFN = D::NFN, NQF = D::NQF;
  constexpr int NT = L::NT, QC = L::QC, CS = L::CS, IT = L::IT;
  extern __shared__ __align__(16) double smem[];
  double* const sS = smem;                   // NM*NM (GS: none)
  double* sC = sS + L::S_;                   // NQ*4*CS
  double* sD = sC + L::C_;                   // QC*25*DS   [qq][st][i]
  double* sW = sD + L::DD_;                  // NN*5
  double* sTR = sW + NN * 5;                 // 4*NFN*5
  double* sPF = sTR + 4 * NFN * 5;           // 4*NQF*FS
  double* sFP = sPF + 4 * NQF * D::FS;       // NQF*FS
  double* sQW = sFP + NQF * D::FS;           // NQ
  double* sFW = sQW + NQ;                    // NQF
  double* sHW = sFW + NQF;                   // 4*NQF*25 (all tiles)
  double* sCol = sHW + 4 * NQF * 25;         // 2*NM (GS: none)
  double* sRow = sCol + (L::GS ? 0 : 2 * NM);
  double* sGeo = sRow + (L::GS ? 0 : 2 * NM);   // 32
  int* sRows = (int*)(sGeo + 32);
  int* sFid = sRows + 4 * NFN;
  int* sTid = sFid + 4;
  int* sBnd = sTid + 4 * NFN;
  int* sQ = sBnd + 4;                        // NM
  int* sQi = sQ + NM;                        // NM
  int* sFlag = sQi + NM;
  double* sQn = (double*)(((size_t)(sFlag + 4) + 15) & ~(size_t)15);   // NN*15 (viscous)
  const double* __restrict__ Bt = g.B;
  const double gam = g.gamma;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 4 * NQF * NFN; i += NT) sPF[(i / NFN) * D::FS + i % NFN] = g.pf[i];
  for (int i = tid; i < NQF * NFN; i += NT) sFP[(i / NFN) * D::FS + i % NFN] = g.fphi[i];
  for (int i = tid; i < NQ; i += NT) sQW[i] = g.qw[i];
  for (int i = tid; i < NQF; i += NT) sFW[i] = g.fw[i];
  for (int i = tid; i < 4 * NFN; i += NT) sRows[i] = g.rows[i];
  // padding lanes of C (st >= 25) stay zero
  for (int i = tid; i < L::C_; i += NT) sC[i] = 0.0;

#ifdef MHDG_RES_TIMING
  long long tl = clock64();
#define LIN_T(k) do { const long long t_ = clock64(); if (tid == 0) atomicAdd(&g_res_clk[k], (unsigned long long)(t_ - tl)); tl = t_; } while (0)
#else
#define LIN_T(k) do { } while (0)
#endif
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    double* const S = L::GS ? sinv + (size_t)e * NM * NM : sS;
    __syncthreads();
    const int en = e + gridDim.x;
    for (int i = tid; i < NN * 5; i += NT) sW[i] = w[(size_t)e * NN * 5 + i];
    if (VISC)
      for (int i = tid; i < NN * 15; i += NT) sQn[i] = qn[(size_t)e * NN * 15 + i];
    // the next macro's inputs towards L2 (its load phase was HBM-latency bound)
    if (MHDG_LIN2_PREFETCH && en < g.E) {
      if (tid < (NN * 5 * 8 + 127) / 128) prefetch_l2(reinterpret_cast<const char*>(w + (size_t)en * NN * 5) + tid * 128);
      if (tid == 32) prefetch_l2(g.fid + en * 4);
      if (tid == 33) prefetch_l2(g.det + en);
      if (tid == 34) prefetch_l2(g.invj + (size_t)en * 9);
      if (tid == 35) prefetch_l2(g.nrm + (size_t)en * 12);
      if (tid == 36) prefetch_l2(g.area + (size_t)en * 4);
      if (tid >= 64 && tid < 64 + (4 * NFN * 4 + 127) / 128)
        prefetch_l2(reinterpret_cast<const char*>(g.tidx + (size_t)en * 4 * NFN) + (tid - 64) * 128);
    }
    if (tid < 4) {
      sFid[tid] = g.fid[e * 4 + tid];
      sBnd[tid] = g.bnd ? g.bnd[e * 4 + tid] : 0;
    }
    for (int i = tid; i < 4 * NFN; i += NT) sTid[i] = g.tidx[(size_t)e * 4 * NFN + i];
    if (tid == 32) sGeo[0] = g.det[e];
    if (tid >= 33 && tid < 42) sGeo[tid - 32] = g.invj[(size_t)e * 9 + tid - 33];
    if (tid >= 42 && tid < 54) sGeo[tid - 32] = g.nrm[(size_t)e * 12 + tid - 42];
    if (tid >= 54 && tid < 58) sGeo[tid - 32] = g.area[(size_t)e * 4 + tid - 54];
    __syncthreads();
    for (int i = tid; i < 4 * NFN * 5; i += NT) {
      const int k = i / (NFN * 5), j = (i / 5) % NFN, s2 = i % 5;
      sTR[i] = trace[((size_t)sFid[k] * NFN + sTid[k * NFN + j]) * 5 + s2];
    }
    LIN_T(0);
    // ---- pointwise duals for all volume quadrature points
    for (int it = tid; it < NQ * 5; it += NT)
      lin2_volume_item<P, VISC, false>(g, vg, it, sW, sQn, sQW, sGeo, weight, sC);
    __syncthreads();
    LIN_T(1);
    // ---- S volume blocks on the tensor cores
    for (int pass = 0; pass < L::NPASS; ++pass) {
    double acc[L::PPW][IT][2];
#pragma unroll
    for (int c = 0; c < L::PPW; ++c)
#pragma unroll
      for (int jt = 0; jt < IT; ++jt) acc[c][jt][0] = acc[c][jt][1] = 0.0;
    for (int ch = 0; ch < L::NCH; ++ch) {
      const int q0 = ch * QC;
      // stage 1: warp w -> chunk point qq = w: D[qq][st][i]
      if (warp < QC) {
        const int qq = warp, q = q0 + qq;
        const int kk = lane & 3, r8 = lane >> 2;
#pragma unroll
        for (int itl = 0; itl < IT; ++itl) {
          const int i = itl * 8 + r8;
          const double a = (q < NQ && i < NN) ? __ldg(Bt + ((size_t)q * 4 + kk) * NN + i) : 0.0;
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            const double b = (q < NQ && (!L::GS || nt * 8 + r8 < 25))
                                 ? sC[(size_t)q * 4 * CS + LIN2_CI(kk, nt * 8 + r8)] : 0.0;
            double c2[2] = {0.0, 0.0};
            dmma_8x8x4(c2, a, b);
            const int ii = itl * 8 + r8, st0 = nt * 8 + (lane & 3) * 2;
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (st0 + h < 25) sD[((size_t)qq * 25 + st0 + h) * L::DS + ii] = c2[h];
          }
        }
      }
      __syncthreads();
      // stage 2: pairs (st, i-tile) owned by this warp, j-tiles in registers
#pragma unroll
      for (int ks = 0; ks < QC / 4; ++ks) {
        const int qq = ks * 4 + (lane & 3), q = q0 + qq;
        double bf[IT];
#pragma unroll
        for (int jt = 0; jt < IT; ++jt) {
          const int j = jt * 8 + (lane >> 2);
          bf[jt] = (q < NQ && j < NN) ? __ldg(Bt + ((size_t)q * 4 + 3) * NN + j) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < L::PPW; ++c) {
          const int pr = warp + L::NW * (pass * L::PPW + c);
          if (pr < L::NPAIR) {
            const int st = pr / IT, itl = pr % IT;
            const double a = sD[((size_t)qq * 25 + st) * L::DS + itl * 8 + (lane >> 2)];
#pragma unroll
            for (int jt = 0; jt < IT; ++jt) dmma_8x8x4(acc[c][jt], a, bf[jt]);
          }
        }
      }
      // the previous macro's S must have left shared memory before the
      // scatter below overwrites it: waited for here, a load phase, the volume
      // duals and the DMMA chunks after its bulk store was issued (at the loop
      // top the wait exposed the store's drain), and published by the barrier
      if (!L::GS && ch == L::NCH - 1 && tid == 0) bulk_wait_read();
      __syncthreads();
    }
    // scatter the accumulators into S[(i,s)][(j,t)]
#pragma unroll
    for (int c = 0; c < L::PPW; ++c) {
      const int pr = warp + L::NW * (pass * L::PPW + c);
      if (pr < L::NPAIR) {
        const int st = pr / IT, itl = pr % IT, s2 = st / 5, t = st % 5;
        const int i = itl * 8 + (lane >> 2);
#pragma unroll
        for (int jt = 0; jt < IT; ++jt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = jt * 8 + (lane & 3) * 2 + h;
            if (i < NN && j < NN) S[(i * 5 + s2) * NM + j * 5 + t] = acc[c][jt][h];
          }
      }
    }
    }   // pass
    // ---- face tiles: hw, hhat, hh tensors of all four tiles in one pass,
    //      then the S face blocks tile by tile (fixed accumulation order)
    __syncthreads();
    LIN_T(2);
    if (MHDG_LIN2_PREFETCH && en < g.E && tid >= NT - 4 * NFN) {   // the next macro's trace rows towards L2 (last warps: they run fewer face items)
      const int i = tid - (NT - 4 * NFN), k = i / NFN;
      const int f = g.fid[en * 4 + k], t2 = g.tidx[(size_t)en * 4 * NFN + i];
      prefetch_l2(trace + ((size_t)f * NFN + t2) * 5);
    }
    for (int it4 = tid; it4 < 4 * NQF * 10; it4 += NT) {
#ifdef MHDG_RES_TIMING
      const long long tr0 = clock64();
#endif
      lin2_face_item<P, VISC, FK>(g, vg, e, it4, sW, sTR, sQn, sPF, sFP, sRows, sGeo, sBnd, ptc, hw_out, hhat_out,
                                  hh_out, sHW);
#ifdef MHDG_RES_TIMING
      if (tid == 0) atomicAdd(&g_res_clk[26 + min(it4 / NT, 2)], (unsigned long long)(clock64() - tr0));
#endif
    }
    __syncthreads();
    LIN_T(3);
#ifndef MHDG_LIN2_FACE_FMA
#define MHDG_LIN2_FACE_FMA 1
#endif
#if MHDG_LIN2_FACE_FMA
    // face weights folded into the staged hw rows once (fw_q area_k hw_q),
    // so each face-block term is one FMA with pf_i pf_j (was mul, mul, add)
    for (int i = tid; i < 4 * NQF * 25; i += NT) {
      const int k = i / (NQF * 25), q = (i / 25) % NQF;
      sHW[i] *= sFW[q] * sGeo[22 + k];
    }
#endif
#ifndef MHDG_LIN2_FACE_DMMA
#define MHDG_LIN2_FACE_DMMA 1
#endif
#if MHDG_LIN2_FACE_DMMA && MHDG_LIN2_FACE_FMA
    // S face blocks on the tensor cores: rows = the face's node pairs (i, j),
    // K = face points, N = (s, t); A = pf_i pf_j formed on the fly, B = the
    // staged weighted hw rows.  A warp takes (pair tile, half of the N tiles)
    // units; every S entry of a face gets exactly one term, so the adds of a
    // face do not collide (the former thread-per-(pair, s) FMA loop was
    // bound by its shared-memory loads: 18k of the kernel's 98k cycles per
    // macro at k = 3).
    for (int k = 0; k < 4; ++k) {
      __syncthreads();
      const double* sHWk = sHW + k * NQF * 25;
      constexpr int WMT = (NFN * NFN + 7) / 8, WKS = (NQF + 3) / 4;
      const int kq = lane & 3, nr = lane >> 2;
      // two units per pass: four independent DMMA chains per warp
      for (int u0 = warp; u0 < 2 * WMT; u0 += MHDG_LIN2_FB_PAIR * L::NW) {
        int ia[2], ja[2], nh[2];
        bool rowok[2];
        double c[2][2][2];
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const int u = u0 + uu * L::NW;
          const int ija = (u >> 1) * 8 + nr;
          nh[uu] = u & 1;
          rowok[uu] = uu < MHDG_LIN2_FB_PAIR && u < 2 * WMT && ija < NFN * NFN;
          ia[uu] = rowok[uu] ? ija / NFN : 0;
          ja[uu] = rowok[uu] ? ija % NFN : 0;
          c[uu][0][0] = c[uu][0][1] = c[uu][1][0] = c[uu][1][1] = 0.0;
        }
        const bool two = MHDG_LIN2_FB_PAIR > 1 && u0 + L::NW < 2 * WMT;   // warp-uniform
#pragma unroll
        for (int ks = 0; ks < WKS; ++ks) {
          const int qa = ks * 4 + kq;
          const double* pf = sPF + (k * NQF + (qa < NQF ? qa : 0)) * D::FS;
          double av[2], bv[2][2];
#pragma unroll
          for (int uu = 0; uu < 2; ++uu) {
            av[uu] = (rowok[uu] && qa < NQF) ? pf[ia[uu]] * pf[ja[uu]] : 0.0;
#pragma unroll
            for (int ntl = 0; ntl < 2; ++ntl) {
              const int n = (nh[uu] * 2 + ntl) * 8 + nr;
              bv[uu][ntl] = (qa < NQF && n < 25) ? sHWk[qa * 25 + n] : 0.0;
            }
          }
          dmma_8x8x4(c[0][0], av[0], bv[0][0]);
          dmma_8x8x4(c[0][1], av[0], bv[0][1]);
          if (two) {
            dmma_8x8x4(c[1][0], av[1], bv[1][0]);
            dmma_8x8x4(c[1][1], av[1], bv[1][1]);
          }
        }
#pragma unroll
        for (int uu = 0; uu < 2; ++uu)
          if (rowok[uu]) {
            const int rb = sRows[k * NFN + ia[uu]] * 5, cb = sRows[k * NFN + ja[uu]] * 5;
#pragma unroll
            for (int ntl = 0; ntl < 2; ++ntl)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int st = (nh[uu] * 2 + ntl) * 8 + kq * 2 + h;
                if (st < 25) S[(rb + st / 5) * NM + cb + st % 5] += c[uu][ntl][h];
              }
          }
      }
    }
#else
    for (int k = 0; k < 4; ++k) {
      __syncthreads();
      const double* sHWk = sHW + k * NQF * 25;
      const double ar = sGeo[22 + k];
      // face block of S: thread = (node pair, row component), 5 accumulators
      for (int o = tid; o < NFN * NFN * 5; o += NT) {
        const int ij = o / 5, s2 = o % 5;
        const int i = ij / NFN, j = ij % NFN;
        double acc2[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int q = 0; q < NQF; ++q) {
          const double* pf = sPF + (k * NQF + q) * D::FS;
#if MHDG_LIN2_FACE_FMA
          const double pij = pf[i] * pf[j];
#pragma unroll
          for (int t = 0; t < 5; ++t) acc2[t] = fma(sHWk[q * 25 + s2 * 5 + t], pij, acc2[t]);
          (void)ar;
#else
          const double ci = (sFW[q] * ar) * pf[i], pj = pf[j];
#pragma unroll
          for (int t = 0; t < 5; ++t) acc2[t] += (ci * sHWk[q * 25 + s2 * 5 + t]) * pj;
#endif
        }
        const int r = sRows[k * NFN + i] * 5 + s2, c = sRows[k * NFN + j] * 5;
#pragma unroll
        for (int t = 0; t < 5; ++t) S[r * NM + c + t] += acc2[t];
      }
    }
#endif
    // ---- S (row-major) to the S^-1 buffer with one TMA bulk store (80 KB at
    //      k = 3); the Gauss-Jordan inverts it in place (GS: already there)
    if (!L::GS) {
      fence_proxy_async();
      __syncthreads();
      LIN_T(4);
      if (tid == 0) bulk_s2g(sinv + (size_t)e * NM * NM, S, (uint32_t)(NM * NM * sizeof(double)));
    }
  }
  if (!L::GS && tid == 0) bulk_wait_all();
}

// ===========================================================================
// K4 (factor): face-block preconditioner  (assembly.py:994-1026, 736-752)
// ===========================================================================
template <int P, int NT>
struct PreSmem {
  using D = Dims<P>;
  static constexpr int NB = D::NB;
  // side block on DMMA: C[(i,j)][(s,t)] = sum_q W[(i,j)][q] hh[q][(s,t)],
  // W[(i,j)][q] = facet_w[q] fphi[q][i] fphi[q][j] (a reference table,
  // lane-swizzled A fragments), times the side's area
  static constexpr int WMT = (D::NFN * D::NFN + 7) / 8, WKS = (D::NQF + 3) / 4, WNT = 4;
  static constexpr int WA = WMT * WKS * 32;
  static constexpr size_t bytes = ((size_t)NB * NB + D::NQF * 25 + D::NQF * D::NFN + 4 * (NB + 16) + D::NQF + WA) * 8 +
                                  ((size_t)D::NFN + 2 * NB + 2) * 4;
};

template <int P, int NT, bool INV = true>   // INV false: store the assembled block row-major
__global__ void __launch_bounds__(NT)
k_precond_factor(Geo g, int n_faces, const double* __restrict__ hh, const double* __restrict__ hh_rem,
                 const int* __restrict__ tidx_rem, const double* __restrict__ area_rem,
                 double* __restrict__ pinv, unsigned long long* status, int* n_unsym) {
  using D = Dims<P>;
  constexpr int NB = D::NB;
  constexpr int TR = NT >= 128 ? 16 : 8, TC = NT / TR;
  extern __shared__ __align__(16) double smem[];
  double* A = smem;                      // NB*NB
  double* sHH = A + NB * NB;             // NQF*25
  double* sFP = sHH + D::NQF * 25;       // NQF*NFN
  double* sCol = sFP + D::NQF * D::NFN;  // 2*NPR
  double* sRow = sCol + 2 * (NB + 16);   // 2*NPC
  double* sFw = sRow + 2 * (NB + 16);    // NQF
  double* sWA = sFw + D::NQF;            // WA
  int* sT = (int*)(sWA + PreSmem<P, NT>::WA);   // NFN
  int* sQ = sT + D::NFN;                 // NB
  int* sQi = sQ + NB;                    // NB
  int* sFlag = sQi + NB;                 // 2
  using PS = PreSmem<P, NT>;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < D::NQF * D::NFN; i += NT) sFP[i] = g.fphi[i];
  for (int i = tid; i < PS::WA; i += NT) {   // [mt][ks][lane]
    const int ln = i % 32, ks = (i / 32) % PS::WKS, mt = i / (32 * PS::WKS);
    const int ij = mt * 8 + (ln >> 2), q = ks * 4 + (ln & 3);
    sWA[i] = (ij < D::NFN * D::NFN && q < D::NQF)
                 ? (g.fw[q] * g.fphi[q * D::NFN + ij / D::NFN]) * g.fphi[q * D::NFN + ij % D::NFN] : 0.0;
  }
  for (int f = blockIdx.x; f < n_faces; f += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < NB * NB; i += NT) A[i] = 0.0;
    for (int side = 0; side < 2; ++side) {
      const int st = g.fsides[f * 2 + side];
      if (st == -1) continue;
      __syncthreads();
      if (st >= 0) {
        const int e = st / 4, k = st % 4;
        for (int i = tid; i < D::NQF * 25; i += NT)   // (25, NQF) per side -> [q][u]
          sHH[(i % D::NQF) * 25 + i / D::NQF] = hh[((size_t)st * D::NQF) * 25 + i];
        for (int i = tid; i < D::NFN; i += NT) sT[i] = g.tidx[((size_t)e * 4 + k) * D::NFN + i];
        if (tid == 0) sFw[0] = g.area[(size_t)e * 4 + k];
      } else {  // remote side of a halo face (partitioned runs)
        const int r = -2 - st;
        for (int i = tid; i < D::NQF * 25; i += NT)
          sHH[(i % D::NQF) * 25 + i / D::NQF] = hh_rem[(size_t)r * D::NQF * 25 + i];
        for (int i = tid; i < D::NFN; i += NT) sT[i] = tidx_rem[(size_t)r * D::NFN + i];
        if (tid == 0) sFw[0] = area_rem[r];
      }
      __syncthreads();
      // side block on the FP64 tensor cores: every ((i,j), (s,t)) is a
      // distinct entry of A, so the warps add their tiles without atomics
      const double area = sFw[0];
      for (int job = warp; job < PS::WMT * PS::WNT; job += NT / 32) {
        const int mt = job / PS::WNT, nt = job % PS::WNT;
        double c[2] = {0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < PS::WKS; ++ks) {
          const int q = ks * 4 + (lane & 3), n = nt * 8 + (lane >> 2);
          const double b = (q < D::NQF && n < 25) ? sHH[q * 25 + n] : 0.0;
          dmma_8x8x4(c, sWA[(mt * PS::WKS + ks) * 32 + lane], b);
        }
        const int ij = mt * 8 + (lane >> 2);
        if (ij < D::NFN * D::NFN) {
          const int i = ij / D::NFN, j = ij % D::NFN;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int st2 = nt * 8 + (lane & 3) * 2 + h2;
            if (st2 < 25) A[(sT[i] * 5 + st2 / 5) * NB + sT[j] * 5 + st2 % 5] += area * c[h2];
          }
        }
      }
    }
    __syncthreads();
    // symmetry statistic (the reference logs the count of non-SPD/non-symmetric
    // blocks): max |a| and max |a - a^T| over the whole CTA
    {
      double amax = 0.0, dmax = 0.0;
      for (int idx = tid; idx < NB * NB; idx += NT) {
        const int r = idx / NB, c = idx % NB;
        amax = fmax(amax, fabs(A[idx]));
        if (c > r) dmax = fmax(dmax, fabs(A[idx] - A[c * NB + r]));
      }
      for (int off = 16; off > 0; off >>= 1) {
        amax = fmax(amax, __shfl_down_sync(0xffffffffu, amax, off));
        dmax = fmax(dmax, __shfl_down_sync(0xffffffffu, dmax, off));
      }
      if ((tid & 31) == 0) {
        sCol[tid >> 5] = amax;
        sRow[tid >> 5] = dmax;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < NT / 32; ++w) {
          amax = fmax(amax, sCol[w]);
          dmax = fmax(dmax, sRow[w]);
        }
        if (!(dmax <= 1e-12 * fmax(1.0, amax))) atomicAdd(n_unsym, 1);
      }
    }
    __syncthreads();
    if (!INV) {   // inverted afterwards by k_gj_blocked<NB>
      for (int i = tid; i < NB * NB; i += NT) pinv[(size_t)f * NB * NB + i] = A[i];
      continue;
    }
    using G = GJDims<NB, TR, TC>;
    double wr[G::RA][G::CB];
    {
      const int tr = tid / TC, tc = tid % TC;
#pragma unroll
      for (int a = 0; a < G::RA; ++a)
#pragma unroll
        for (int b = 0; b < G::CB; ++b) {
          const int r = tr + TR * a, c = tc + TC * b;
          wr[a][b] = (tid < TR * TC && r < NB && c < NB) ? A[r * NB + c] : 0.0;
        }
      __syncthreads();
      bool ok0 = gj_inverse_reg<NB, TR, TC>(wr, sCol, sRow, sQ, sFlag);
#pragma unroll
      for (int a = 0; a < G::RA; ++a)
#pragma unroll
        for (int b = 0; b < G::CB; ++b) {
          const int r = tr + TR * a, c = tc + TC * b;
          if (tid < TR * TC && r < NB && c < NB) A[r * NB + c] = wr[a][b];
        }
      __syncthreads();
      sFlag[1] = ok0;
    }
    bool ok = gj_store_colmajor<NB, NT>(A, sQ, sQi, pinv + (size_t)f * NB * NB) && (sFlag[1] != 0);
    if (!ok && tid == 0) report(status, 0, 0, f);
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
// z_e = S_e^-1 g_e (column-major S^-1); neg: g = -gin (condensed rhs).
// Thread (macro slot, row) per output; small systems (NM < NT / 2) take
// several macros per block so every thread streams a row.
template <int NM>
struct LocalSolveCfg {
  static constexpr int NT = NM <= 128 ? 128 : 192;
  static constexpr int MB = NM <= NT / 2 ? NT / NM : 1;   // macros per block iteration
};

template <int NM, int NT>
__global__ void __launch_bounds__(NT)
k_local_solve(int E, const double* __restrict__ sinv, const double* __restrict__ gin, int neg,
              double* __restrict__ z) {
  constexpr int MB = LocalSolveCfg<NM>::MB;
  __shared__ double sg[MB * NM];
  const int ml = threadIdx.x / NM, rr = threadIdx.x % NM;
  pdl_wait();   // nothing precedes the wait but index arithmetic
  for (int e0 = blockIdx.x * MB; e0 < E; e0 += gridDim.x * MB) {
    const int nm = min(MB, E - e0);
    __syncthreads();
    for (int i = threadIdx.x; i < nm * NM; i += NT) sg[i] = neg ? -gin[(size_t)e0 * NM + i] : gin[(size_t)e0 * NM + i];
    __syncthreads();
    if constexpr (MB > 1) {
      if (ml >= nm) continue;
    }
    const int e = e0 + (MB > 1 ? ml : 0);
    const double* A = sinv + (size_t)e * NM * NM;
    const double* g = sg + (MB > 1 ? ml * NM : 0);
    for (int r = (MB > 1 ? rr : threadIdx.x); r < NM; r += (MB > 1 ? NM : NT)) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int c = 0;
      for (; c + 3 < NM; c += 4) {
        a0 += __ldcs(A + (size_t)(c + 0) * NM + r) * g[c + 0];
        a1 += __ldcs(A + (size_t)(c + 1) * NM + r) * g[c + 1];
        a2 += __ldcs(A + (size_t)(c + 2) * NM + r) * g[c + 2];
        a3 += __ldcs(A + (size_t)(c + 3) * NM + r) * g[c + 3];
      }
      for (; c < NM; ++c) a0 += __ldcs(A + (size_t)c * NM + r) * g[c];
      z[(size_t)e * NM + r] = (a0 + a1) + (a2 + a3);
    }
  }
}

// Register-blocked face kernels: one thread per (macro slot, tile, face
// point); its 25-entry tensor rows for the NEXT macro batch are prefetched
// straight into registers (no shared-memory staging of the 12.8 KB/macro
// tensors), and every shared-memory read feeds a 5-wide register block.
template <int P>
struct Face2 {
  using D = Dims<P>;
  static constexpr int NI = 4 * D::NQF;                        // items per macro
  static constexpr int NT = 128;
  static constexpr int EB = (NT / NI) > 0 ? (NT / NI) : 1;    // macros per iteration
  static constexpr int IPT = (EB * NI + NT - 1) / NT;          // items per thread
  static constexpr int NX = 4 * D::NFN * 5;
  static constexpr int XPT = (EB * NX + NT - 1) / NT;
  static constexpr int ZPT = (EB * D::NM + NT - 1) / NT;
  static constexpr int META = 4 + 4 * D::NFN;
  static constexpr int MPT = (EB * (META + 4) + NT - 1) / NT;
  // phase-2 test contraction on DMMA: M tiles over the NFN face nodes, K
  // steps over the NQF face points; A fragments (phi_face per tile for
  // MODE 0, fphi for MODE 1) lane-swizzled in shared memory
  static constexpr int TMT = (D::NFN + 7) / 8;
  static constexpr int TKS = (D::NQF + 3) / 4;
  static constexpr int AF = 4 * TMT * TKS * 32;
  static constexpr int doubles = 4 * D::NQF * D::FS + D::NQF * D::FS + D::NQF + EB * (NX + D::NM + 2 * NI * 5 + NX) +
                                 3 * EB * 4 + AF;
  static constexpr int ints = 4 * D::NFN + 3 * D::NN + 3 * EB * META;
  static constexpr size_t bytes = (size_t)doubles * 8 + ints * 4;
};

#ifndef MHDG_FACE_MINB_LOW
#define MHDG_FACE_MINB_LOW 4   // resident CTAs per SM of the k <= 2 face-in kernel (measured 3 / 4 / 5: k = 1 matvec 0.655 / 0.640 / 0.678 ms, k = 2 1.645 / 1.622 / 1.621)
#endif
template <int P, int MODE>   // MODE 0: g = -A_vh x (+ -r_w); 1: y += A_hh x + A_hv z
__global__ void __launch_bounds__(128, (P <= 2 && MODE == 0) ? MHDG_FACE_MINB_LOW : 3)
k_face2(Geo g, int mode, const double* __restrict__ tenA, const double* __restrict__ tenB,
        const double* __restrict__ x, const double* __restrict__ zin, const double* __restrict__ r_w,
        double* __restrict__ out) {
  using D = Dims<P>;
  using F2 = Face2<P>;
  constexpr int NM = D::NM, NFN = D::NFN, NQF = D::NQF, NN = D::NN, NI = F2::NI, NX = F2::NX, META = F2::META;
  constexpr int NT = F2::NT, EB = F2::EB;
  const bool use_x = (MODE == 0) || mode == 0;
  const bool use_b = (MODE == 1) && mode == 0;
  extern __shared__ __align__(16) double smem[];
  double* sPF = smem;
  double* sFP = sPF + 4 * NQF * D::FS;
  double* sFW = sFP + NQF * D::FS;
  double* sX = sFW + NQF;                 // EB*NX
  double* sZ = sX + EB * NX;              // EB*NM
  double* sA = sZ + EB * NM;              // EB*NI*5
  double* sB = sA + EB * NI * 5;          // EB*NI*5
  double* sT = sB + EB * NI * 5;          // EB*NX
  double* sAr = sT + EB * NX;             // 3*EB*4
  double* sAF = sAr + 3 * EB * 4;         // AF
  int* sRows = (int*)(sAF + F2::AF);
  int* sNF = sRows + 4 * NFN;
  int* sMeta = sNF + 3 * NN;              // 3*EB*META
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // [k][mt][ks][lane]: lane = 4 r + c holds F[q = 4 ks + c][j = 8 mt + r]
  for (int i = tid; i < F2::AF; i += NT) {
    const int ln = i % 32, ks = (i / 32) % F2::TKS, mt = (i / (32 * F2::TKS)) % F2::TMT,
              k = i / (32 * F2::TKS * F2::TMT);
    const int j = mt * 8 + (ln >> 2), q = ks * 4 + (ln & 3);
    double v = 0.0;
    if (q < NQF && j < NFN) v = (MODE == 0) ? g.pf[(k * NQF + q) * NFN + j] : g.fphi[q * NFN + j];
    sAF[i] = v;
  }
  for (int i = tid; i < 4 * NQF * NFN; i += NT) sPF[(i / NFN) * D::FS + i % NFN] = g.pf[i];
  for (int i = tid; i < NQF * NFN; i += NT) sFP[(i / NFN) * D::FS + i % NFN] = g.fphi[i];
  for (int i = tid; i < NQF; i += NT) sFW[i] = g.fw[i];
  for (int i = tid; i < 4 * NFN; i += NT) sRows[i] = g.rows[i];
  for (int i = tid; i < 3 * NN; i += NT) sNF[i] = g.nodef[i];
  const int G = gridDim.x * EB;
  auto meta_elem = [&](int e0, int i, int& iv, double& dv) {   // i over EB*(META+4)
    const int m = i / (META + 4), r = i % (META + 4), e = e0 + m;
    if (e >= g.E) return;
    if (r < 4) iv = g.fid[e * 4 + r];
    else if (r < META) iv = g.tidx[(size_t)e * 4 * NFN + r - 4];
    else dv = g.area[(size_t)e * 4 + r - META];
  };
  auto meta_put = [&](int slot, int i, int iv, double dv) {
    const int m = i / (META + 4), r = i % (META + 4);
    if (r < META) sMeta[(slot * EB + m) * META + r] = iv;
    else sAr[(slot * EB + m) * 4 + r - META] = dv;
  };
  const int e00 = blockIdx.x * EB;
  for (int c = 0; c < 2; ++c)
    for (int i = tid; i < EB * (META + 4); i += NT) {
      int iv = 0;
      double dv = 0.0;
      meta_elem(e00 + c * G, i, iv, dv);
      meta_put(c, i, iv, dv);
    }
  __syncthreads();
  double rA[F2::IPT][25], rB[F2::IPT][25], rX[F2::XPT], rZ[F2::ZPT], rMd[F2::MPT];
  int rMi[F2::MPT];
  auto prefetch = [&](int e0, int slot) {
#pragma unroll
    for (int c = 0; c < F2::IPT; ++c) {
      const int it = tid + c * NT, m = it / NI, e = e0 + m;
      if (it < EB * NI && e < g.E) {
        // (E, 4, 25, NQF): entry u of consecutive face points is contiguous
        const int kq = it % NI;
        const size_t tb = ((size_t)e * 4 + kq / NQF) * 25 * NQF + kq % NQF;
#pragma unroll
        for (int u = 0; u < 25; ++u) rA[c][u] = __ldcs(tenA + tb + u * NQF);
        if (use_b)
#pragma unroll
          for (int u = 0; u < 25; ++u) rB[c][u] = __ldcs(tenB + tb + u * NQF);
      }
    }
    if (use_x) {
#pragma unroll
      for (int c = 0; c < F2::XPT; ++c) {
        const int i = tid + c * NT, m = i / NX, r = i % NX, e = e0 + m;
        if (i < EB * NX && e < g.E) {
          const int* mt = sMeta + (slot * EB + m) * META;
          const int k = r / (NFN * 5), j = (r / 5) % NFN, s2 = r % 5;
          rX[c] = x[((size_t)mt[k] * NFN + mt[4 + k * NFN + j]) * 5 + s2];
        }
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int c = 0; c < F2::ZPT; ++c) {
        const int i = tid + c * NT, m = i / NM, e = e0 + m;
        if (i < EB * NM && e < g.E) rZ[c] = zin[(size_t)e * NM + i % NM];
      }
    }
  };
  // before the wait: reference tables and face metadata (fid, tidx, area) into
  // shared memory only; prefetch() (reads x / zin / hhat) runs after it
  pdl_wait();
  if (e00 < g.E) prefetch(e00, 0);
  int slot = 0;
  for (int e0 = e00; e0 < g.E; e0 += G, slot = (slot + 1) % 3) {
    const int e1 = e0 + G, e2 = e0 + 2 * G;
    const int s1 = (slot + 1) % 3, s2s = (slot + 2) % 3;
    const int nm = min(EB, g.E - e0);
    __syncthreads();
    if (use_x) {
#pragma unroll
      for (int c = 0; c < F2::XPT; ++c) {
        const int i = tid + c * NT;
        if (i < EB * NX) sX[i] = rX[c];
      }
    }
    if (MODE == 1) {
#pragma unroll
      for (int c = 0; c < F2::ZPT; ++c) {
        const int i = tid + c * NT;
        if (i < EB * NM) sZ[i] = rZ[c];
      }
    }
    __syncthreads();
    // ---- phase 1: per (slot m, tile k, point q): 5-vectors at the point
    if (e2 < g.E) {
#pragma unroll
      for (int c = 0; c < F2::MPT; ++c) {
        const int i = tid + c * NT;
        rMi[c] = 0;
        rMd[c] = 0.0;
        if (i < EB * (META + 4)) meta_elem(e2, i, rMi[c], rMd[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < F2::IPT; ++c) {
      const int it = tid + c * NT, m = it / NI, kq = it % NI, k = kq / NQF, q = kq % NQF;
      if (it < EB * NI && m < nm) {
        const double fwq = sFW[q] * sAr[(slot * EB + m) * 4 + k];
        double xq[5] = {0, 0, 0, 0, 0}, zq[5] = {0, 0, 0, 0, 0};
        if (use_x) {
          const double* fp = sFP + q * D::FS;
          const double* xs = sX + m * NX + k * NFN * 5;
#pragma unroll
          for (int j = 0; j < NFN; ++j) {
            const double f = fp[j];
#pragma unroll
            for (int t = 0; t < 5; ++t) xq[t] += f * xs[j * 5 + t];
          }
        }
        if (MODE == 1) {
          const double* pf = sPF + kq * D::FS;
          const double* zs = sZ + m * NM;
#pragma unroll
          for (int j = 0; j < NFN; ++j) {
            const double f = pf[j];
            const int row = sRows[k * NFN + j];
#pragma unroll
            for (int t = 0; t < 5; ++t) zq[t] += f * zs[row * 5 + t];
          }
        }
#pragma unroll
        for (int s2 = 0; s2 < 5; ++s2) {
          double a = 0.0, b = 0.0;
#pragma unroll
          for (int t = 0; t < 5; ++t) {
            a += rA[c][s2 * 5 + t] * (MODE == 0 ? xq[t] : zq[t]);
            if (use_b) b += rB[c][s2 * 5 + t] * xq[t];
          }
          // MODE 1 tests A_hv z and A_hh x with the same fphi rows: one sum
          sA[it * 5 + s2] = use_b ? fwq * a + fwq * b : fwq * a;
        }
      }
    }
    // next batch: tensor rows / trace values / z into the same registers
    if (e1 < g.E) prefetch(e1, s1);
    __syncthreads();
    // ---- phase 2: per (slot m, tile k) on DMMA: C[j][s] = sum_q F[q][j] V[q][s]
    for (int job = warp; job < nm * 4; job += NT / 32) {
      const int m = job / 4, k = job % 4;
      const double* V = sA + (m * NI + k * NQF) * 5;
      const double* af = sAF + (MODE == 0 ? k * F2::TMT * F2::TKS * 32 : 0);
      const int kq_ = lane & 3, n_ = lane >> 2;
      double c[F2::TMT][2];
#pragma unroll
      for (int t = 0; t < F2::TMT; ++t) c[t][0] = c[t][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < F2::TKS; ++ks) {
        const int q = ks * 4 + kq_;
        const double vb = (n_ < 5 && q < NQF) ? V[q * 5 + n_] : 0.0;
#pragma unroll
        for (int t = 0; t < F2::TMT; ++t) dmma_8x8x4(c[t], af[(t * F2::TKS + ks) * 32 + lane], vb);
      }
      const int* mt = sMeta + (slot * EB + m) * META;
#pragma unroll
      for (int t = 0; t < F2::TMT; ++t)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int j = t * 8 + n_, s2 = kq_ * 2 + h2;
          if (j < NFN && s2 < 5) {
            if (MODE == 0) sT[m * NX + (k * NFN + j) * 5 + s2] = c[t][h2];
            else atomicAdd(&out[((size_t)mt[k] * NFN + mt[4 + k * NFN + j]) * 5 + s2], c[t][h2]);
          }
        }
    }
    if (MODE == 0) {
      __syncthreads();
      for (int o = tid; o < nm * NM; o += NT) {
        const int m = o / NM, r = o % NM, i = r / 5, s2 = r % 5;
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int kj = sNF[i * 3 + c];
          if (kj < 0) break;
          v += sT[m * NX + kj * 5 + s2];
        }
        const size_t gi = (size_t)(e0 + m) * NM + r;
        out[gi] = (mode == 0) ? -v : (-r_w[gi] + (-v));
      }
    }
    if (e2 < g.E) {
#pragma unroll
      for (int c = 0; c < F2::MPT; ++c) {
        const int i = tid + c * NT;
        if (i < EB * (META + 4)) meta_put(s2s, i, rMi[c], rMd[c]);
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
  pdl_wait();   // first instruction: r is the predecessor's output
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

// entropy identity monitor, face part (assembly.py:649-672 with
// fluxes.py:245-255): per side tile k and face point q of every macro
//   r = (v(u_hat) - v(u)) . F^(u, u_hat; n) - (psi_n(u_hat) - psi_n(u)),
//   psi_n(u) = rho V . n, summed with face_w = fw_q area_k; per-block
// partials (the caller reduces them in a fixed order).
template <int P, int NT>
__global__ void __launch_bounds__(NT)
k_entropy_faces(Geo g, const double* __restrict__ w, const double* __restrict__ tr,
                double* __restrict__ partial) {
  using D = Dims<P>;
  __shared__ double red[NT];
  const double gam = g.gamma;
  double acc = 0.0;
  for (int e = blockIdx.x; e < g.E; e += gridDim.x) {
    for (int t = threadIdx.x; t < 4 * D::NQF; t += NT) {
      const int k = t / D::NQF, q = t % D::NQF;
      double wq[5] = {0, 0, 0, 0, 0}, wh[5] = {0, 0, 0, 0, 0};
      const int f = g.fid[e * 4 + k];
      for (int i = 0; i < D::NFN; ++i) {
        const double a = g.pf[(k * D::NQF + q) * D::NFN + i];
        const double b = g.fphi[q * D::NFN + i];
        const double* wi = w + ((size_t)e * D::NN + g.rows[k * D::NFN + i]) * 5;
        const double* ti = tr + ((size_t)f * D::NFN + g.tidx[((size_t)e * 4 + k) * D::NFN + i]) * 5;
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          wq[s] += a * wi[s];
          wh[s] += b * ti[s];
        }
      }
      double u[5], uh[5], n[3];
      to_conservative(wq, g.form, gam, u);
      to_conservative(wh, g.form, gam, uh);
      for (int a = 0; a < 3; ++a) n[a] = g.nrm[((size_t)e * 4 + k) * 3 + a];
      double fh[5], v[5], vh[5];
      numerical_flux(g.kind, u, uh, n, gam, fh);
      entropy_vars(u, gam, v);
      entropy_vars(uh, gam, vh);
      double r = 0.0;
#pragma unroll
      for (int s = 0; s < 5; ++s) r += (vh[s] - v[s]) * fh[s];
      const double psi = (u[1] * n[0] + u[2] * n[1]) + u[3] * n[2];
      const double psih = (uh[1] * n[0] + uh[2] * n[1]) + uh[3] * n[2];
      r -= psih - psi;
      acc += (g.fw[q] * g.area[e * 4 + k]) * r;
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

// sum over nodes of v(state) . r, v = state (entropy formulation) or
// entropy_vars(state) (conservative): the left side of the identity
__global__ void k_entropy_dot(int64_t n, int form, double gam, const double* __restrict__ x,
                              const double* __restrict__ r, double* __restrict__ partial) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v[5];
    if (form == 1) {
#pragma unroll
      for (int s = 0; s < 5; ++s) v[s] = x[i * 5 + s];
    } else {
      double u[5];
#pragma unroll
      for (int s = 0; s < 5; ++s) u[s] = x[i * 5 + s];
      entropy_vars(u, gam, v);
    }
#pragma unroll
    for (int s = 0; s < 5; ++s) acc += v[s] * r[i * 5 + s];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int sft = 128; sft > 0; sft >>= 1) {
    if (threadIdx.x < sft) red[threadIdx.x] += red[threadIdx.x + sft];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

}  // namespace mhdg
