// mhdg_macro_host.cuh -- context setup and entry points of the m > 1 operator
// (kernels in mhdg_macro.cuh).  Included at the end of mhdg_capi.cu; every C
// entry point forwards here when ctx->m > 1.  Supported (m, p): (2, 1..3),
// (3, 1): the orders of S (5 nc) and of the face blocks (5 nt) then have
// batched Gauss-Jordan instantiations.  Inviscid, periodic.
#pragma once

static mhdg_ctx* mm_create(const mhdg_tables* t, int device, int* err) {
  const int P = t->p, m = t->m;
  const bool ok = (m == 2 && P >= 1 && P <= 3) || (m == 3 && P == 1);
  if (!ok || t->has_visc || t->freestream || !t->scatter || !t->trace_ptr || !t->face_ptr) {
    *err = MHDG_INVALID_CONFIG;
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) { *err = MHDG_CUDA_ERROR; return nullptr; }
  mhdg_ctx* c = new mhdg_ctx();
  c->device = device;
  c->m = m;
  c->p = P;
  c->E = t->n_macros;
  c->F = t->n_faces;
  c->nn = t->nc;      // macro nodes: the size of w rows (E, nc, 5)
  c->nfn = t->nt;     // trace nodes per face: the size of trace rows (F, nt, 5)
  c->nq = t->nq;
  c->nqf = t->nqf;
  c->n_owned = t->n_faces;
  c->visc = 0;
  c->launches = 0;
  c->d_scratch = nullptr;
  c->scratch_bytes = 0;
  cudaDeviceGetAttribute(&c->n_sms, cudaDevAttrMultiProcessorCount, device);
  {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    c->smem_optin = optin > 0 ? (size_t)optin : 48 * 1024;
  }
  memset(&c->geo, 0, sizeof(c->geo));
  memset(&c->vg, 0, sizeof(c->vg));
  const size_t E = t->n_macros, F = t->n_faces;
  const int nsub = t->n_sub, nst = t->n_st, NN = t->nn, NQ = t->nq, NFN = t->nfn, NQF = t->nqf;
  MGeo& g = c->mg;
  memset(&g, 0, sizeof(g));
  g.E = (int)E;
  g.F = (int)F;
  g.nsub = nsub;
  g.nst = nst;
  g.nc = t->nc;
  g.nt = t->nt;
  g.form = t->formulation;
  g.kind = t->flux_kind;
  g.gamma = t->gamma;
  g.phi = upload(c, t->phi, (size_t)NQ * NN, err);
  g.dphi = upload(c, t->dphi, (size_t)NQ * NN * 3, err);
  g.qw = upload(c, t->quad_wts, NQ, err);
  g.pf = upload(c, t->phi_face, (size_t)nst * NQF * NFN, err);
  g.fphi = upload(c, t->fphi, (size_t)NQF * NFN, err);
  g.fw = upload(c, t->facet_wts, NQF, err);
  g.scatter = upload_i64(c, t->scatter, (size_t)nsub * NN, err);
  g.rows = upload_i64(c, t->face_rows, (size_t)nst * NFN, err);
  g.det = upload(c, t->sub_det_all, E * nsub, err);
  g.invj = upload(c, t->sub_inv_jac_all, E * nsub * 9, err);
  g.nrm = upload(c, t->face_normals, E * nst * 3, err);
  g.area = upload(c, t->face_area, E * nst, err);
  g.fid = upload_i64(c, t->face_id_st, E * nst, err);
  g.tidx = upload_i64(c, t->trace_idx, E * nst * NFN, err);
  g.tptr = upload_i64(c, t->trace_ptr, F * t->nt + 1, err);
  g.tlist = upload_i64(c, t->trace_list, E * nst * NFN, err);
  g.fptr = upload_i64(c, t->face_ptr, F + 1, err);
  g.flist = upload_i64(c, t->face_list, E * nst, err);
  c->geo.E = (int)E;
  c->geo.F = (int)F;
  c->geo.form = t->formulation;
  c->geo.kind = t->flux_kind;
  c->geo.gamma = t->gamma;
  c->d_status = (unsigned long long*)dalloc(c, sizeof(unsigned long long) * 4, err);
  c->d_unsym = (int*)dalloc(c, sizeof(int) * 4, err);
  c->d_partial = (double*)dalloc(c, sizeof(double) * (2 * RED_BLOCKS * 5 + 64), err);
  c->d_tmp_trace = (double*)dalloc(c, sizeof(double) * F * t->nt * 5, err);
  c->d_fb = (int*)dalloc(c, sizeof(int) * (2 + std::max(E, F)), err);
  if (c->d_fb) cudaMemset(c->d_fb, 0, 2 * sizeof(int));
  c->d_gbuf = (double*)dalloc(c, sizeof(double) * E * t->nc * 5, err);
  c->d_zbuf = (double*)dalloc(c, sizeof(double) * E * t->nc * 5, err);
  c->d_cb = (double*)dalloc(c, sizeof(double) * E * nst * NFN * 5, err);
  if (*err != MHDG_OK) {
    mhdg_destroy(c);
    return nullptr;
  }
  return c;
}

static void mm_lin_sizes(const mhdg_ctx* c, int64_t sizes[6]) {
  const int64_t nm = 5 * (int64_t)c->mg.nc, nb = 5 * (int64_t)c->mg.nt;
  sizes[0] = (int64_t)c->E * nm * nm;
  sizes[1] = sizes[2] = sizes[3] = (int64_t)c->E * c->mg.nst * c->nqf * 25;
  sizes[4] = (int64_t)c->F * nb * nb;
  sizes[5] = 1;
}

static int mm_grid(mhdg_ctx* c, int items) { return std::max(1, std::min(items, c->n_sms * 8)); }

template <class Fn>
static int mm_by_p(mhdg_ctx* c, Fn&& fn) {
  switch (c->p) {
    case 1: return fn(std::integral_constant<int, 1>{});
    case 2: return fn(std::integral_constant<int, 2>{});
    default: return fn(std::integral_constant<int, 3>{});
  }
}

static int mm_gather_into(mhdg_ctx* c, int mode, const double* a, double* out, cudaStream_t s) {
  const int n = c->F * c->mg.nt;
  mm_gather<<<mm_grid(c, (n * 5 + 255) / 256), 256, 0, s>>>(n, c->mg.tptr, c->mg.tlist, c->d_cb, mode, a, out);
  c->launches++;
  CK(cudaGetLastError());
  return MHDG_OK;
}

static int mm_residual_entry(mhdg_ctx* c, const double* w, const double* trace, int has_stage, double alpha,
                             const double* offset, int check, double* r_w, double* r_trace, cudaStream_t s) {
  CK(cudaMemsetAsync(c->d_status, 0xff, sizeof(unsigned long long), s));
  const size_t smem = (size_t)(2 * c->mg.nc * 5 + c->nq * 20) * 8;
  int rc = mm_by_p(c, [&](auto pc) -> int {
    constexpr int P = decltype(pc)::value;
    if (set_smem(mm_residual<P>, smem)) return MHDG_CUDA_ERROR;
    mm_residual<P><<<mm_grid(c, c->E), 128, smem, s>>>(c->mg, w, trace, has_stage, alpha, offset, check, r_w,
                                                      c->d_cb, c->d_status);
    return MHDG_OK;
  });
  if (rc) return rc;
  c->launches++;
  CK(cudaGetLastError());
  return mm_gather_into(c, 0, nullptr, r_trace, s);
}

static int mm_volume_states_entry(mhdg_ctx* c, const double* w, double* out, cudaStream_t s) {
  CK(cudaMemsetAsync(c->d_status, 0xff, sizeof(unsigned long long), s));
  const int64_t n = (int64_t)c->E * c->mg.nsub * c->nq;
  mm_by_p(c, [&](auto pc) -> int {
    constexpr int P = decltype(pc)::value;
    mm_volume_states<P><<<mm_grid(c, (int)((n + 127) / 128)), 128, 0, s>>>(c->mg, w, out, c->d_status);
    return 0;
  });
  c->launches++;
  CK(cudaGetLastError());
  return MHDG_OK;
}

static int mm_integrals_entry(mhdg_ctx* c, const double* w, double* out_host, cudaStream_t s) {
  double* part = c->d_partial;
  double* res = c->d_partial + 2 * RED_BLOCKS * 5;
  const int nb = RED_BLOCKS;
  mm_by_p(c, [&](auto pc) -> int {
    constexpr int P = decltype(pc)::value;
    mm_integrals<P><<<nb, 128, 0, s>>>(c->mg, w, part);
    return 0;
  });
  k_reduce_rows<<<1, 32, 0, s>>>(nb, 5, part, res);
  c->launches += 2;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_host, res, 5 * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return MHDG_OK;
}

// in-place batched inverse of row-major N x N blocks -> column-major:
// shared-memory lookahead Gauss-Jordan when it fits, else the blocked
// kernel with its working matrix in an L2-resident global slab per CTA
template <int N>
static int mm_invert(mhdg_ctx* c, int nmat, double* mats, unsigned long long* status, cudaStream_t s, int slot) {
  if constexpr (GJLA2<N, (N >= 64 ? MHDG_GJ_NWT : MHDG_GJ_NWT_SMALL), (N >= 64 ? MHDG_GJ_NPW : MHDG_GJ_NPW_SMALL)>::bytes <=
                200 * 1024) {
    return gj_lookahead<N>(c, nmat, mats, status, s, slot);
  } else if (MHDG_GJ_GA && N <= 200) {
    // global-slab lookahead kernel while two slabs per SM stay L2-resident
    // (N = 175: 3x faster than the blocked kernel; N = 420: 10% slower)
    c->launches++;
    return gj_lookahead_ga<N>(c, nmat, mats, status, s, slot);
  } else {
    using GB = GJB<N>;
    const size_t gsm = GB::bytes_gm;
    if (set_smem(k_gj_blocked<N, true>, gsm)) return MHDG_CUDA_ERROR;
    // two CTAs per SM even when their slabs exceed L2 (N = 420: capping the
    // grid to L2-resident slabs measured 2.2x slower, 3.0 vs 1.35 s)
    const int ggrid = grid_for(c, nmat, std::min(2, occ(k_gj_blocked<N, true>, GB::NT, gsm)));
    const size_t slabs = (size_t)ggrid * GB::slab * sizeof(double);
    if (slabs > c->scratch_bytes) {
      if (c->d_scratch) cudaFree(c->d_scratch);
      c->d_scratch = nullptr;
      if (cudaMalloc(&c->d_scratch, slabs) != cudaSuccess) return MHDG_OUT_OF_MEMORY;
      c->scratch_bytes = slabs;
    }
    k_gj_blocked<N, true><<<ggrid, GB::NT, gsm, s>>>(nmat, mats, status, c->d_scratch);
    c->launches++;
    CK(cudaGetLastError());
    return MHDG_OK;
  }
}

static int mm_invert_any(mhdg_ctx* c, int N, int nmat, double* mats, unsigned long long* status, cudaStream_t s,
                         int slot) {
  switch (N) {
    case 30: return mm_invert<30>(c, nmat, mats, status, s, slot);
    case 50: return mm_invert<50>(c, nmat, mats, status, s, slot);
    case 75: return mm_invert<75>(c, nmat, mats, status, s, slot);
    case 100: return mm_invert<100>(c, nmat, mats, status, s, slot);
    case 140: return mm_invert<140>(c, nmat, mats, status, s, slot);
    case 175: return mm_invert<175>(c, nmat, mats, status, s, slot);
    case 420: return mm_invert<420>(c, nmat, mats, status, s, slot);
    default: return MHDG_INVALID_CONFIG;
  }
}

static int mm_linearize_entry(mhdg_ctx* c, const double* w, const double* trace, double alpha, double ptc,
                              const mhdg_lin_buffers* L, mhdg_status* st, cudaStream_t s) {
  CK(cudaMemsetAsync(c->d_status, 0xff, 2 * sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(c->d_unsym, 0, sizeof(int), s));
  const double weight = alpha + ptc;
  const size_t smem = (size_t)(c->mg.nc * 5 + c->nq * 100) * 8;
  int rc = mm_by_p(c, [&](auto pc) -> int {
    constexpr int P = decltype(pc)::value;
    if (set_smem(mm_linearize<P>, smem)) return MHDG_CUDA_ERROR;
    mm_linearize<P><<<mm_grid(c, c->E), 128, smem, s>>>(c->mg, w, trace, weight, ptc, L->sinv, L->hw, L->hhat,
                                                       L->hh);
    mm_precond_blk<P><<<mm_grid(c, c->F), 128, 0, s>>>(c->mg, L->hh, L->pinv, c->d_unsym);
    return MHDG_OK;
  });
  if (rc) return rc;
  c->launches += 2;
  CK(cudaGetLastError());
  rc = mm_invert_any(c, 5 * c->mg.nc, c->E, L->sinv, c->d_status, s, 0);
  if (rc) return rc;
  rc = mm_invert_any(c, 5 * c->mg.nt, c->F, L->pinv, c->d_status + 1, s, 1);
  if (rc) return rc;
  return fetch_lin_status(c, st, s);
}

static int mm_gemv_entry(mhdg_ctx* c, int nmat, int N, const double* A, const double* x, double* y,
                         cudaStream_t s) {
  const size_t smem = (size_t)N * 8;
  const int nt = std::min(512, (N + 31) / 32 * 32);
  const int per_sm = std::max(1, 2048 / nt);
  mm_gemv<<<std::max(1, std::min(nmat, c->n_sms * per_sm)), nt, smem, s>>>(nmat, N, A, x, y);
  c->launches++;
  CK(cudaGetLastError());
  return MHDG_OK;
}

// condensed operator: mode 0 matvec, 1 condensed rhs, 2 recover
static int mm_condensed(mhdg_ctx* c, int mode, const mhdg_lin_buffers* L, const double* x, const double* r_w,
                        const double* r_trace, double* out, double* d_w, cudaStream_t s) {
  const int NM = 5 * c->mg.nc;
  const size_t fsm = (size_t)(c->mg.nc * 5 + c->nqf * 5) * 8;
  // local right-hand side: matvec -A_vh x, rhs -r_w, recover -r_w - A_vh d
  const double* xin = mode == 1 ? nullptr : x;
  const double* rin = mode == 0 ? nullptr : r_w;
  int rc = mm_by_p(c, [&](auto pc) -> int {
    constexpr int P = decltype(pc)::value;
    if (set_smem(mm_face_in<P>, fsm)) return MHDG_CUDA_ERROR;
    mm_face_in<P><<<mm_grid(c, c->E), 128, fsm, s>>>(c->mg, L->hhat, xin, rin, -1.0, c->d_gbuf);
    return MHDG_OK;
  });
  if (rc) return rc;
  c->launches++;
  rc = mm_gemv_entry(c, c->E, NM, L->sinv, c->d_gbuf, mode == 2 ? d_w : c->d_zbuf, s);
  if (rc || mode == 2) return rc;
  rc = mm_by_p(c, [&](auto pc) -> int {
    constexpr int P = decltype(pc)::value;
    mm_face_out<P><<<mm_grid(c, c->E * c->mg.nst), 128, 0, s>>>(c->mg, L->hh, L->hw, mode == 0 ? x : nullptr,
                                                                c->d_zbuf, c->d_cb);
    return MHDG_OK;
  });
  if (rc) return rc;
  c->launches++;
  CK(cudaGetLastError());
  // matvec: y = A_hh x + A_hv z ; rhs: b = -r^ - A_hv S^-1 (-r_w)
  return mode == 0 ? mm_gather_into(c, 0, nullptr, out, s) : mm_gather_into(c, 2, r_trace, out, s);
}
