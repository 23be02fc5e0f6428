// mhdg_krylov.cuh -- device-resident condensed solve: the reference's
// solve_condensed (solver.py:121-170) = flexible GMRES(restart) whose
// preconditioner is an inner GMRES(inner_iters) sweep preconditioned by the
// face-block solve, run as ONE CUDA graph with conditional WHILE / IF nodes:
// no host round trip between Arnoldi steps, restart cycles or inner sweeps.
//
// Control flow of one FGMRES level (solver.py:42-118), all on the device:
//
//   x = 0; r = b; rr = r.r; decide(first)        norm_b, zero-rhs exit
//   WHILE go:                                     restart cycles
//     WHILE cyc:                                  Arnoldi columns j
//       vin = V_j; zout = P(vin)                  P: inner level or face solve
//       w = A zout; Z_j = zout
//       MGS(V, j, w) -> H[:, j], V_{j+1}          one cooperative kernel
//       givens(j) -> cs, sn, g; break tests       sets cyc
//     y = H[:k,:k]^-1 g[:k]; x += Z^T y           back substitution
//     r = b - A x; rr = r.r; decide               sets go (rel <= tol,
//                                                 iteration cap, stagnation)
//
// The outer level's P is the inner level's program followed by an IF node:
// when the inner sweep never updated x, z = face_solve(v) (solver.py:153-154).
// Scalars follow the reference's IEEE operations (Givens rotations and the
// triangular solve without FMA contraction, a correctly rounded hypot);
// vector reductions are the library's fixed-order deterministic ones.
//
// The graph bakes in the linearization's buffer pointers: it is rebuilt when
// mhdg_krylov_solve sees a different mhdg_lin_buffers (one capture + one
// instantiation, ~ms), and reused across Newton iterations otherwise.
#pragma once

#include <cooperative_groups.h>

namespace mhdg_kr {

namespace cg = cooperative_groups;

struct LevelState {
  double norm_b, beta, rel, prev_rel, tol, rr;
  int total, max_iters, restart, m, j, k, go, cyc, converged, updated;
  int inner_sum;  // outer level: inner iterations accumulated over the solve
  int gtest;      // the last column ended the cycle on the Arnoldi residual test
  int ncyc;       // restart cycles finished in this solve
  int ax_ok;      // L.t holds H y of the (single) cycle: A x = V_{k+1} t
};

struct Level {  // device pointers of one level (passed by value to kernels)
  LevelState* st;
  double *H, *cs, *sn, *g, *y;   // H column-major, column j at H + j * (R + 1)
  double *Hraw, *t;              // H before the rotations; t = Hraw[:k+1,:k] y
  double *V, *Z, *vin, *zout, *w, *x, *r, *tmp;
  const double* b;
  int R;
};

// ---- scalar kernels (one thread) -----------------------------------------

// IEEE operations without contraction: the reference evaluates these on
// numpy float64 scalars, one rounding per operation
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// hypot(a, b), correctly rounded except in rare double-rounding ties (the
// reference calls Python's math.hypot, which is correctly rounded in the
// same sense): the sum of squares carried in double-double, one Newton
// correction of the square root
__device__ double hypot_cr(double a, double b) {
  double x = fabs(a), y = fabs(b);
  if (x < y) { const double t = x; x = y; y = t; }
  if (x == 0.0) return 0.0;
  if (isinf(x)) return x;
  // scale by a power of two so the squares neither overflow nor underflow
  int ex;
  frexp(x, &ex);
  const double sc = ldexp(1.0, -ex);
  x *= sc;
  y *= sc;
  const double xx = x * x, xx_lo = fma(x, x, -xx);
  const double yy = y * y, yy_lo = fma(y, y, -yy);
  double s = xx + yy;
  const double bb = s - xx;
  double s_lo = (xx - (s - bb)) + (yy - bb) + xx_lo + yy_lo;
  const double t = s + s_lo;
  s_lo = s_lo - (t - s);
  s = t;
  double h = sqrt(s);
  const double rem = fma(-h, h, s) + s_lo;
  h = h + rem / (2.0 * h);
  return ldexp(h, ex);
}

__global__ void k_kr_reset(Level L, int outer) {
  LevelState* s = L.st;
  s->total = 0;
  s->prev_rel = INFINITY;
  s->converged = 0;
  s->updated = 0;
  s->go = 0;
  s->cyc = 0;
  s->k = 0;
  s->j = 0;
  s->gtest = 0;
  s->ncyc = 0;
  s->ax_ok = 0;
  if (outer) s->inner_sum = 0;
}

__global__ void k_kr_set(cudaGraphConditionalHandle h, unsigned int v) { cudaGraphSetConditional(h, v); }

// solver.py:55-80: first = 1 also sets norm_b (r = b on the first pass)
__global__ void k_kr_decide(Level L, int first, cudaGraphConditionalHandle h_go) {
  LevelState* s = L.st;
  int go = 0;
  if (first) s->norm_b = sqrt(s->rr);
  if (s->norm_b == 0.0) {  // zero right-hand side: x = 0, converged
    s->rel = 0.0;
    s->converged = 1;
  } else {
    s->beta = sqrt(s->rr);
    const double rel = s->beta / s->norm_b;
    s->rel = rel;
    if (rel <= s->tol) {
      s->converged = 1;
    } else if (s->total >= s->max_iters) {
      // unconverged
    } else if (rel >= s->prev_rel * (1 - 1e-12)) {
      // stagnation over a restart cycle (raise_on_stagnation=False)
    } else {
      s->prev_rel = rel;
      s->m = min(s->restart, s->max_iters - s->total);
      s->j = 0;
      s->k = 0;
      L.g[0] = s->beta;
      go = 1;
    }
  }
  s->go = go;
  s->cyc = go;
  cudaGraphSetConditional(h_go, go);
}

// solver.py:95-115 for column j (H[:, j] holds the MGS coefficients)
__global__ void k_kr_givens(Level L, cudaGraphConditionalHandle h_cyc) {
  LevelState* s = L.st;
  const int j = s->j, ld = L.R + 1;
  double* h = L.H + (int64_t)j * ld;
  const double hnorm = h[j + 1];
  for (int i = 0; i <= j + 1; ++i) L.Hraw[(int64_t)j * ld + i] = h[i];
  for (int i = 0; i < j; ++i) {
    const double t = add(mul(L.cs[i], h[i]), mul(L.sn[i], h[i + 1]));
    h[i + 1] = add(mul(-L.sn[i], h[i]), mul(L.cs[i], h[i + 1]));
    h[i] = t;
  }
  const double denom = hypot_cr(h[j], h[j + 1]);
  int cyc = 1;
  s->gtest = 0;
  if (denom == 0.0) {
    cyc = 0;  // Krylov space exhausted without progress on this column
  } else {
    L.cs[j] = h[j] / denom;
    L.sn[j] = h[j + 1] / denom;
    h[j] = denom;
    h[j + 1] = 0.0;
    L.g[j + 1] = mul(-L.sn[j], L.g[j]);
    L.g[j] = mul(L.g[j], L.cs[j]);
    s->total += 1;
    s->k = j + 1;
    const int gt = fabs(L.g[j + 1]) / s->norm_b <= s->tol;
    s->gtest = gt;
    if (gt || hnorm <= 1e-300) cyc = 0;
    else if (j + 1 >= s->m) cyc = 0;
    else s->j = j + 1;
  }
  s->cyc = cyc;
  cudaGraphSetConditional(h_cyc, cyc);
}

// y = H[:k,:k]^-1 g[:k] (upper triangular, column-oriented back substitution
// as BLAS trsv) and the updated flag (solver.py:116-118)
__global__ void k_kr_trisolve(Level L) {
  LevelState* s = L.st;
  const int k = s->k, ld = L.R + 1;
  if (k <= 0) return;
  for (int i = 0; i < k; ++i) L.y[i] = L.g[i];
  for (int c = k - 1; c >= 0; --c) {
    const double yc = L.y[c] / L.H[(int64_t)c * ld + c];
    L.y[c] = yc;
    for (int i = 0; i < c; ++i) L.y[i] = sub(L.y[i], mul(L.H[(int64_t)c * ld + i], yc));
  }
  s->updated = 1;
}

// End of an inner sweep's cycle without the true-residual matvec
// (mhdg_krylov_params.inner_true_residual = 0).  solver.py:62-72 after the
// cycle: r = b - A x, then return x when rel <= tol or total >= max_iters.
// On the iteration cap x is returned whatever r is, so the matvec is dead
// work (exact); when the cycle ended on |g_k| / |b| <= tol, that Arnoldi
// estimate is the residual norm of x in exact arithmetic and stands in for
// it.  Breakdown exits (hnorm tiny, zero rotation) keep the true residual.
__global__ void k_kr_cycle_end(Level L, cudaGraphConditionalHandle h_true, cudaGraphConditionalHandle h_go) {
  LevelState* s = L.st;
  const bool skip = s->k > 0 && (s->gtest || s->total >= s->max_iters);
  // A x of this sweep from its Arnoldi relation A Z = V H (x = Z y, one
  // cycle from x = 0): t = H y over the k + 1 basis vectors
  if (skip && s->ncyc == 0) {
    const int k = s->k, ld = L.R + 1;
    for (int i = 0; i <= k; ++i) {
      double a = 0.0;
      for (int c = (i > 0 ? i - 1 : 0); c < k; ++c) a += L.Hraw[(int64_t)c * ld + i] * L.y[c];
      L.t[i] = a;
    }
    s->ax_ok = 1;
  }
  s->ncyc += 1;
  if (skip) {
    const double rel = fabs(L.g[s->k]) / s->norm_b;
    s->rel = rel;
    s->converged = rel <= s->tol;
    s->go = 0;
    s->cyc = 0;
    cudaGraphSetConditional(h_go, 0u);
  }
  cudaGraphSetConditional(h_true, skip ? 0u : 1u);
}

// inner sweep finished: count its iterations into the outer level and arm
// the IF node "inner never updated x -> face solve" (solver.py:150-154)
__global__ void k_kr_inner_done(Level inner, Level outer, cudaGraphConditionalHandle h_noupd,
                                cudaGraphConditionalHandle h_ax, cudaGraphConditionalHandle h_mv, int reuse) {
  outer.st->inner_sum += inner.st->total;
  cudaGraphSetConditional(h_noupd, inner.st->updated ? 0u : 1u);
  // w = A z from the sweep's Arnoldi relation, or by the operator
  const unsigned ax = (reuse && inner.st->updated && inner.st->ax_ok) ? 1u : 0u;
  cudaGraphSetConditional(h_ax, ax);
  cudaGraphSetConditional(h_mv, 1u - ax);
}

// w = V_{k+1} t (A x of the inner sweep, k and t read on the device)
__global__ void k_kr_lincomb(int64_t n, const double* __restrict__ V, const double* __restrict__ t,
                             const LevelState* __restrict__ s, double* __restrict__ w) {
  const int k = s->k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r <= k; ++r) acc += V[(int64_t)r * n + i] * t[r];
    w[i] = acc;
  }
}

// ---- vector kernels --------------------------------------------------------

__global__ void k_kr_row_copy(int64_t n, double* base, const int* __restrict__ jp, int to_row, double* vec) {
  double* row = base + (int64_t)(*jp) * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (to_row) row[i] = vec[i];
    else vec[i] = row[i];
  }
}

// V_0 = r / beta, vin = V_0
__global__ void k_kr_start_basis(int64_t n, const double* __restrict__ r, const LevelState* __restrict__ s,
                                 double* __restrict__ v0) {
  if (!s->go) return;
  const double beta = s->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v0[i] = r[i] / beta;
}

// x += Z^T y over the k columns of the cycle (k read on the device)
__global__ void k_kr_combine(int64_t n, const double* __restrict__ Z, const double* __restrict__ y,
                             const LevelState* __restrict__ s, double* __restrict__ x) {
  const int k = s->k;
  if (k <= 0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < k; ++r) acc += Z[(int64_t)r * n + i] * y[r];
    x[i] = x[i] + acc;
  }
}

// z = x_inner when the inner sweep updated it
__global__ void k_kr_select(int64_t n, const LevelState* __restrict__ s, const double* __restrict__ x,
                            double* __restrict__ z) {
  if (!s->updated) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = x[i];
}

__device__ __forceinline__ double kr_block_sum(double v, double* sh) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += sh[i];
  return r;
}

// every block reduces the same partials in the same order -> same scalar
__device__ __forceinline__ double kr_reduce(const double* __restrict__ part, int nblk, double* sh) {
  double v = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) v += part[b];
  const double r = kr_block_sum(v, sh);
  if (threadIdx.x == 0) sh[32] = r;
  __syncthreads();
  const double out = sh[32];
  __syncthreads();
  return out;
}

// Modified Gram-Schmidt of w against V_0..V_j (solver.py:101-106), j read on
// the device: one cooperative kernel, one grid barrier per basis vector.
// Step i reduces <V_i, w>, updates w and forms the partials of the next
// product in the same pass.  Writes H[0..j+1, j] and, if ||w|| > 1e-300,
// V_{j+1} = w / ||w|| (also into vin_next, the next column's input).
__global__ void __launch_bounds__(256)
k_kr_mgs(int64_t n, double* __restrict__ V, double* __restrict__ w, LevelState* __restrict__ s,
         double* __restrict__ H, int ld, double* __restrict__ part) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[40];
  const int j = s->j;
  const int nb = gridDim.x;
  double* hcol = H + (int64_t)j * ld;
  double* pa = part;
  double* pb = part + nb;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
  double v = 0.0;
  for (int64_t i = i0; i < n; i += st) v += V[i] * w[i];
  double r = kr_block_sum(v, sh);
  if (threadIdx.x == 0) pa[blockIdx.x] = r;
  grid.sync();
  for (int q = 0; q <= j; ++q) {
    const double h = kr_reduce(pa, nb, sh);
    if (blockIdx.x == 0 && threadIdx.x == 0) hcol[q] = h;
    const double* vq = V + (int64_t)q * n;
    const double* vn = (q < j) ? V + (int64_t)(q + 1) * n : nullptr;
    double acc = 0.0;
    for (int64_t i = i0; i < n; i += st) {
      const double wn = w[i] - h * vq[i];
      w[i] = wn;
      acc += (vn ? vn[i] : wn) * wn;
    }
    r = kr_block_sum(acc, sh);
    if (threadIdx.x == 0) pb[blockIdx.x] = r;
    grid.sync();
    double* t = pa;
    pa = pb;
    pb = t;
  }
  const double hn = sqrt(kr_reduce(pa, nb, sh));
  if (blockIdx.x == 0 && threadIdx.x == 0) hcol[j + 1] = hn;
  if (!(hn > 1e-300)) return;
  double* vnew = V + (int64_t)(j + 1) * n;
  for (int64_t i = i0; i < n; i += st) vnew[i] = w[i] / hn;
}

__global__ void __launch_bounds__(256)
k_kr_dot(int64_t n, const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ part,
         double* __restrict__ out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[40];
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v += x[i] * y[i];
  const double r = kr_block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
  grid.sync();
  if (blockIdx.x == 0) {
    const double t = kr_reduce(part, gridDim.x, sh);
    if (threadIdx.x == 0) out[0] = t;
  }
}

}  // namespace mhdg_kr

// ---------------------------------------------------------------------------
// engine object
// ---------------------------------------------------------------------------
struct mhdg_krylov {
  mhdg_ctx* c;
  int device;
  mhdg_krylov_params prm;
  int64_t n;
  int coop_grid;
  double* part;  // 2 x coop_grid partials
  mhdg_kr::Level L[2];  // 0 outer, 1 inner
  double* b;     // engine-owned right-hand side
  mhdg_krylov_stats* d_stats;
  mhdg_lin_buffers lin;  // pointers the graph was built for
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  int built;
  cudaStream_t cap;  // capture stream (non-blocking, private)
};

namespace mhdg_kr {

struct Builder {
  mhdg_krylov* K;
  cudaStream_t s;
  int err;
  // append a captured segment to graph g after node dep (nullptr = root)
  template <class F>
  cudaGraphNode_t seg(cudaGraph_t g, cudaGraphNode_t dep, F&& body) {
    if (err) return nullptr;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { err = 1; return nullptr; }
    const int rc = body(s);
    cudaGraph_t child = nullptr;
    const cudaError_t e = cudaStreamEndCapture(s, &child);
    if (rc || e != cudaSuccess || !child) { err = rc ? rc : 1; return nullptr; }
    cudaGraphNode_t node = nullptr;
    if (cudaGraphAddChildGraphNode(&node, g, dep ? &dep : nullptr, dep ? 1 : 0, child) != cudaSuccess) err = 1;
    cudaGraphDestroy(child);
    return node;
  }
  // conditional node (WHILE / IF) after dep; returns its body graph
  cudaGraphNode_t cond(cudaGraph_t g, cudaGraphNode_t dep, cudaGraphConditionalHandle h,
                       cudaGraphConditionalNodeType type, cudaGraph_t* body) {
    if (err) return nullptr;
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = 1;
    cudaGraphNode_t node = nullptr;
    if (cudaGraphAddNode(&node, g, dep ? &dep : nullptr, dep ? 1 : 0, &p) != cudaSuccess) { err = 1; return nullptr; }
    *body = p.conditional.phGraph_out[0];
    return node;
  }
  cudaGraphConditionalHandle handle(cudaGraph_t g) {
    cudaGraphConditionalHandle h = 0;
    if (!err && cudaGraphConditionalHandleCreate(&h, g, 0, 0) != cudaSuccess) err = 1;
    return h;
  }
};

}  // namespace mhdg_kr

static int kr_grid(mhdg_krylov* K, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)K->c->n_sms * 8));
}

static cudaError_t kr_coop(void (*k)(int64_t, double*, double*, mhdg_kr::LevelState*, double*, int, double*),
                           int grid, cudaStream_t s, int64_t n, double* V, double* w, mhdg_kr::LevelState* st,
                           double* H, int ld, double* part) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, n, V, w, st, H, ld, part);
}

static cudaError_t kr_dot(mhdg_krylov* K, cudaStream_t s, const double* x, const double* y, double* out) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(K->coop_grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mhdg_kr::k_kr_dot, K->n, x, y, K->part, out);
}

// body of one Arnoldi column of level `lv` into graph g (after dep); the
// preconditioner of the outer level is the whole inner program
static cudaGraphNode_t kr_column(mhdg_kr::Builder& B, cudaGraph_t g, int lv, cudaGraphConditionalHandle h_cyc);

// full program of one level (reset .. WHILE go) into graph g after dep
static cudaGraphNode_t kr_level(mhdg_kr::Builder& B, cudaGraph_t g, cudaGraphNode_t dep, int lv) {
  using namespace mhdg_kr;
  mhdg_krylov* K = B.K;
  mhdg_ctx* c = K->c;
  const Level L = K->L[lv];
  const int64_t n = K->n;
  const int gr = kr_grid(K, n);
  // a conditional handle belongs to the graph holding its node; it is set
  // by kernels upstream in that graph or inside its (nested) bodies
  cudaGraphConditionalHandle h_go = B.handle(g);
  // prologue: x = 0, r = b, rr = r.r, decide(first), V_0 = r / beta
  dep = B.seg(g, dep, [&](cudaStream_t s) -> int {
    k_kr_reset<<<1, 1, 0, s>>>(L, lv == 0);
    CK(cudaMemsetAsync(L.x, 0, sizeof(double) * n, s));
    CK(cudaMemcpyAsync(L.r, L.b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    CK(kr_dot(K, s, L.r, L.r, &L.st->rr));
    k_kr_decide<<<1, 1, 0, s>>>(L, 1, h_go);
    k_kr_start_basis<<<gr, 256, 0, s>>>(n, L.r, L.st, L.V);
    CK(cudaGetLastError());
    return 0;
  });
  cudaGraph_t body_go = nullptr;
  dep = B.cond(g, dep, h_go, cudaGraphCondTypeWhile, &body_go);
  if (B.err) return nullptr;
  // restart cycle: cyc = 1; WHILE cyc { column } ; update x ; r = b - A x ; decide
  cudaGraphConditionalHandle h_cyc = B.handle(body_go);
  cudaGraphNode_t d1 = B.seg(body_go, nullptr, [&](cudaStream_t s) -> int {
    k_kr_set<<<1, 1, 0, s>>>(h_cyc, 1u);
    CK(cudaGetLastError());
    return 0;
  });
  cudaGraph_t body_cyc = nullptr;
  cudaGraphNode_t d2 = B.cond(body_go, d1, h_cyc, cudaGraphCondTypeWhile, &body_cyc);
  kr_column(B, body_cyc, lv, h_cyc);
  // update x, then the true residual and the restart decision; the inner
  // sweep skips the latter when its cycle ended on the cap or the Arnoldi test
  cudaGraph_t tail = body_go;
  cudaGraphNode_t d3 = d2;
  if (lv == 1 && !K->prm.inner_true_residual) {
    cudaGraphConditionalHandle h_true = B.handle(body_go);
    d3 = B.seg(body_go, d2, [&](cudaStream_t s) -> int {
      k_kr_trisolve<<<1, 1, 0, s>>>(L);
      k_kr_combine<<<gr, 256, 0, s>>>(n, L.Z, L.y, L.st, L.x);
      k_kr_cycle_end<<<1, 1, 0, s>>>(L, h_true, h_go);
      CK(cudaGetLastError());
      return 0;
    });
    B.cond(body_go, d3, h_true, cudaGraphCondTypeIf, &tail);
    if (B.err) return nullptr;
    d3 = nullptr;
  }
  const bool update_here = tail == body_go;
  B.seg(tail, d3, [&](cudaStream_t s) -> int {
    if (update_here) {
      k_kr_trisolve<<<1, 1, 0, s>>>(L);
      k_kr_combine<<<gr, 256, 0, s>>>(n, L.Z, L.y, L.st, L.x);
      CK(cudaGetLastError());
    }
    int rc = mhdg_matvec(c, &K->lin, L.x, L.tmp, (void*)s);
    if (rc) return rc;
    rc = mhdg_axpby(c, n, 1.0, L.b, -1.0, L.tmp, L.r, (void*)s);
    if (rc) return rc;
    CK(kr_dot(K, s, L.r, L.r, &L.st->rr));
    k_kr_decide<<<1, 1, 0, s>>>(L, 0, h_go);
    k_kr_start_basis<<<gr, 256, 0, s>>>(n, L.r, L.st, L.V);
    CK(cudaGetLastError());
    return 0;
  });
  return dep;
}

static cudaGraphNode_t kr_column(mhdg_kr::Builder& B, cudaGraph_t g, int lv, cudaGraphConditionalHandle h_cyc) {
  using namespace mhdg_kr;
  mhdg_krylov* K = B.K;
  mhdg_ctx* c = K->c;
  const Level L = K->L[lv];
  const int64_t n = K->n;
  const int gr = kr_grid(K, n);
  cudaGraphConditionalHandle h_ax = 0, h_mv = 0;
  bool split_w = false;
  // vin = V_j
  cudaGraphNode_t dep = B.seg(g, nullptr, [&](cudaStream_t s) -> int {
    k_kr_row_copy<<<gr, 256, 0, s>>>(n, L.V, &L.st->j, 0, L.vin);
    CK(cudaGetLastError());
    return 0;
  });
  // zout = P(vin)
  if (lv == 0 && K->prm.inner_precond) {
    const Level I = K->L[1];
    dep = kr_level(B, g, dep, 1);  // inner program: b = outer vin
    cudaGraphConditionalHandle h_noupd = B.handle(g);
    h_ax = B.handle(g);
    h_mv = B.handle(g);
    split_w = true;
    dep = B.seg(g, dep, [&](cudaStream_t s) -> int {
      k_kr_inner_done<<<1, 1, 0, s>>>(I, L, h_noupd, h_ax, h_mv, K->prm.outer_matvec_reuse);
      CK(cudaGetLastError());
      return 0;
    });
    cudaGraph_t body_if = nullptr;
    dep = B.cond(g, dep, h_noupd, cudaGraphCondTypeIf, &body_if);
    if (B.err) return nullptr;
    B.seg(body_if, nullptr, [&](cudaStream_t s) -> int {
      return mhdg_precond(c, &K->lin, L.vin, L.zout, (void*)s);
    });
    dep = B.seg(g, dep, [&](cudaStream_t s) -> int {
      k_kr_select<<<gr, 256, 0, s>>>(n, I.st, I.x, L.zout);
      CK(cudaGetLastError());
      return 0;
    });
  } else {
    dep = B.seg(g, dep, [&](cudaStream_t s) -> int {
      return mhdg_precond(c, &K->lin, L.vin, L.zout, (void*)s);
    });
  }
  // w = A zout: from the inner sweep's Arnoldi relation when it has one
  // (IF h_ax), by the operator otherwise (IF h_mv)
  if (split_w) {
    const Level I = K->L[1];
    cudaGraph_t body_ax = nullptr, body_mv = nullptr;
    dep = B.cond(g, dep, h_ax, cudaGraphCondTypeIf, &body_ax);
    if (B.err) return nullptr;
    B.seg(body_ax, nullptr, [&](cudaStream_t s) -> int {
      k_kr_lincomb<<<gr, 256, 0, s>>>(n, I.V, I.t, I.st, L.w);
      CK(cudaGetLastError());
      return 0;
    });
    dep = B.cond(g, dep, h_mv, cudaGraphCondTypeIf, &body_mv);
    if (B.err) return nullptr;
    B.seg(body_mv, nullptr, [&](cudaStream_t s) -> int {
      return mhdg_matvec(c, &K->lin, L.zout, L.w, (void*)s);
    });
  }
  // Z_j = zout; MGS; Givens (sets cyc)
  return B.seg(g, dep, [&](cudaStream_t s) -> int {
    if (!split_w) {
      const int rc = mhdg_matvec(c, &K->lin, L.zout, L.w, (void*)s);
      if (rc) return rc;
    }
    k_kr_row_copy<<<gr, 256, 0, s>>>(n, L.Z, &L.st->j, 1, L.zout);
    CK(cudaGetLastError());
    CK(kr_coop(k_kr_mgs, K->coop_grid, s, n, L.V, L.w, L.st, L.H, L.R + 1, K->part));
    k_kr_givens<<<1, 1, 0, s>>>(L, h_cyc);
    CK(cudaGetLastError());
    return 0;
  });
}

static int kr_build(mhdg_krylov* K) {
  if (K->built) {
    cudaGraphExecDestroy(K->exec);
    cudaGraphDestroy(K->graph);
    K->built = 0;
  }
  CK(cudaGraphCreate(&K->graph, 0));
  mhdg_kr::Builder B{K, K->cap, 0};
  kr_level(B, K->graph, nullptr, 0);
  if (B.err) {
    cudaGraphDestroy(K->graph);
    return B.err > 1 ? B.err : MHDG_CUDA_ERROR;
  }
  if (cudaGraphInstantiate(&K->exec, K->graph, 0) != cudaSuccess) {
    cudaGraphDestroy(K->graph);
    return MHDG_CUDA_ERROR;
  }
  K->built = 1;
  return MHDG_OK;
}

extern "C" int64_t mhdg_krylov_workspace(const mhdg_ctx* c, const mhdg_krylov_params* prm) {
  const int64_t n = (int64_t)c->F * c->nfn * 5;
  auto level = [&](int R) {
    return (int64_t)(R + 1) * n + (int64_t)R * n + 6 * n  // V, Z, vin zout w x r tmp
           + 2 * (int64_t)(R + 1) * R + 5 * (int64_t)R + 3 + 16;   // H, Hraw, cs sn g y t, state
  };
  return level(prm->restart) + (prm->inner_precond ? level(prm->inner_iters) : 0) + n + 4 +
         2 * (int64_t)c->n_sms * 32;
}

extern "C" mhdg_krylov* mhdg_krylov_create(mhdg_ctx* c, const mhdg_krylov_params* prm, double* workspace,
                                           int64_t workspace_len, int* err) {
  *err = MHDG_OK;
  if (prm->restart < 1 || prm->max_outer < 0 || prm->inner_iters < 1 || !(prm->rel_tol > 0) ||
      !(prm->inner_rtol > 0) || (prm->outer_matvec_reuse && prm->inner_true_residual)) {
    *err = MHDG_INVALID_CONFIG;
    return nullptr;
  }
  if (workspace_len < mhdg_krylov_workspace(c, prm)) {
    *err = MHDG_INVALID_CONFIG;
    return nullptr;
  }
  if (cudaSetDevice(c->device) != cudaSuccess) { *err = MHDG_CUDA_ERROR; return nullptr; }
  mhdg_krylov* K = new mhdg_krylov();
  K->c = c;
  K->device = c->device;
  K->prm = *prm;
  K->n = (int64_t)c->F * c->nfn * 5;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mhdg_kr::k_kr_mgs, 256, 0);
  int per_sm2 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, mhdg_kr::k_kr_dot, 256, 0);
  per_sm = std::max(1, std::min(std::min(per_sm, per_sm2), 4));
  K->coop_grid = c->n_sms * per_sm;
  double* p = workspace;
  const int64_t n = K->n;
  auto take = [&](int64_t cnt) { double* q = p; p += cnt; return q; };
  K->b = take(n);
  K->d_stats = (mhdg_krylov_stats*)take(4);
  K->part = take(2 * (int64_t)c->n_sms * 32);
  for (int lv = 0; lv < (prm->inner_precond ? 2 : 1); ++lv) {
    const int R = lv == 0 ? prm->restart : prm->inner_iters;
    mhdg_kr::Level& L = K->L[lv];
    L.R = R;
    L.st = (mhdg_kr::LevelState*)take(16);
    L.H = take((int64_t)(R + 1) * R);
    L.cs = take(R);
    L.sn = take(R);
    L.g = take(R + 2);
    L.y = take(R);
    L.Hraw = take((int64_t)(R + 1) * R);
    L.t = take(R + 1);
    L.V = take((int64_t)(R + 1) * n);
    L.Z = take((int64_t)R * n);
    L.vin = take(n);
    L.zout = take(n);
    L.w = take(n);
    L.x = take(n);
    L.r = take(n);
    L.tmp = take(n);
  }
  K->L[0].b = K->b;
  if (prm->inner_precond) K->L[1].b = K->L[0].vin;
  // constant scalars of each level
  mhdg_kr::LevelState st[2] = {};
  st[0].tol = prm->rel_tol;
  st[0].restart = prm->restart;
  st[0].max_iters = prm->max_outer;
  st[1].tol = prm->inner_rtol;
  st[1].restart = prm->inner_iters;
  st[1].max_iters = prm->inner_iters;
  for (int lv = 0; lv < (prm->inner_precond ? 2 : 1); ++lv)
    if (cudaMemcpy(K->L[lv].st, &st[lv], sizeof(st[lv]), cudaMemcpyHostToDevice) != cudaSuccess)
      *err = MHDG_CUDA_ERROR;
  if (cudaStreamCreateWithFlags(&K->cap, cudaStreamNonBlocking) != cudaSuccess) *err = MHDG_CUDA_ERROR;
  if (*err) {
    delete K;
    return nullptr;
  }
  return K;
}

// Must run before mhdg_destroy of its context (the Python owner destroys its
// engines first); touches only the engine's own objects and leaves no error
// behind for the next cudaGetLastError of the library.
extern "C" void mhdg_krylov_destroy(mhdg_krylov* K) {
  if (!K) return;
  int cur = -1;
  cudaGetDevice(&cur);
  cudaSetDevice(K->device);
  if (K->built) {
    cudaGraphExecDestroy(K->exec);
    cudaGraphDestroy(K->graph);
  }
  cudaStreamDestroy(K->cap);
  if (cur >= 0) cudaSetDevice(cur);
  cudaGetLastError();
  delete K;
}

// final scalars of the outer level -> stats (device side, copied to host once)
__global__ void k_kr_stats(const mhdg_kr::LevelState* __restrict__ s, int inner, mhdg_krylov_stats* out) {
  out->outer_iterations = s->total;
  out->inner_iterations = inner ? s->inner_sum : 0;
  out->converged = s->converged;
  out->updated = s->updated;
  out->rel_residual = s->rel;
}

extern "C" int mhdg_krylov_solve(mhdg_krylov* K, const mhdg_lin_buffers* lin, const double* b, double* x,
                                 mhdg_krylov_stats* stats, int sync, void* stream) {
  mhdg_ctx* c = K->c;
  cudaStream_t s = S(stream);
  CK(cudaSetDevice(c->device));
  if (!K->built || memcmp(&K->lin, lin, sizeof(*lin)) != 0) {
    K->lin = *lin;
    // the capture stream must not run ahead of work queued on the caller's
    // stream (nothing is executed during capture, so no ordering is needed;
    // the graph is launched on the caller's stream below)
    const int64_t l0 = c->launches;
    const int rc = kr_build(K);
    c->launches = l0;
    if (rc) return rc;
  }
  const int64_t n = K->n;
  CK(cudaMemcpyAsync(K->b, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  CK(cudaGraphLaunch(K->exec, s));
  CK(cudaMemcpyAsync(x, K->L[0].x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  k_kr_stats<<<1, 1, 0, s>>>(K->L[0].st, K->prm.inner_precond, K->d_stats);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(stats, K->d_stats, sizeof(*stats), cudaMemcpyDeviceToHost, s));
  if (sync) CK(cudaStreamSynchronize(s));
  c->launches += 1;
  return MHDG_OK;
}
