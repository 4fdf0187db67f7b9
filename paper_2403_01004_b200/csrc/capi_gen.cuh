// paracycle_b200 C ABI, part of the single translation unit capi.cu (included
// there in order; relies on the declarations of the parts before it).
//
// C ABI: synthetic-input generators (bit-identical to the host recipes of
// paper_2403_01004_b200/configs.py)
#pragma once

// ------------------------------------------------------------------ synthetic inputs
// (configs.py recipes evaluated in HBM; tables are GLOBAL-grid tables)
static int upload_tmp(pc_ctx* c, const double* host, size_t n, double** dev) {
  CUDA_TRY(cudaMalloc(dev, n * sizeof(double)));
  CUDA_TRY(cudaMemcpyAsync(*dev, host, n * sizeof(double), cudaMemcpyHostToDevice, c->s));
  return PC_OK;
}
static const double kSqrt3 = 1.7320508075688772;  // math.sqrt(3.0)

int pc_gen_temperature(pc_field* T, uint64_t seed, int stream, double sigma, const double* prof) {
  field_dep(T);
  if (!T || T->ncomp != 1 || !prof) return fail(PC_E_INVALID, "temperature: scalar field and profile needed");
  pc_grid* g = T->grid;
  pc_ctx* c = g->ctx;
  double* dp = nullptr;
  TRY(upload_tmp(c, prof, (size_t)g->g.n0g, &dp));
  k_gen_temperature<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, T->base(0), stream_key(seed, stream), sigma,
                                                                  dp, kSqrt3);
  c->st.launches++;
  int rc = check_launch("k_gen_temperature");
  cudaStreamSynchronize(c->s);
  cudaFree(dp);
  return rc;
}

int pc_gen_dipole(pc_field* b, uint64_t seed, int stream0, double eps, const double* ir3, const double* c2,
                  const double* st) {
  field_dep(b);
  if (!b || b->ncomp != 3 || !ir3 || !c2 || !st) return fail(PC_E_INVALID, "dipole: 3-component field and tables");
  pc_grid* g = b->grid;
  pc_ctx* c = g->ctx;
  double *d0 = nullptr, *d1 = nullptr, *d2 = nullptr;
  TRY(upload_tmp(c, ir3, (size_t)g->g.n0g, &d0));
  TRY(upload_tmp(c, c2, (size_t)g->g.n1, &d1));
  TRY(upload_tmp(c, st, (size_t)g->g.n1, &d2));
  k_gen_dipole<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, fld(b), stream_key(seed, stream0),
                                                             stream_key(seed, stream0 + 1),
                                                             stream_key(seed, stream0 + 2), eps, d0, d1, d2, kSqrt3);
  c->st.launches++;
  int rc = check_launch("k_gen_dipole");
  cudaStreamSynchronize(c->s);
  cudaFree(d0);
  cudaFree(d1);
  cudaFree(d2);
  return rc;
}

int pc_gen_harmonic(pc_field* v, const double* acc, double checker) {
  field_dep(v);
  if (!v || !acc) return fail(PC_E_INVALID, "harmonic: field and (ncomp, n1, n2) table needed");
  pc_grid* g = v->grid;
  pc_ctx* c = g->ctx;
  double* da = nullptr;
  TRY(upload_tmp(c, acc, (size_t)v->ncomp * g->g.n1 * g->g.n2, &da));
  k_gen_harmonic<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, fld(v), v->ncomp, da, checker);
  c->st.launches++;
  int rc = check_launch("k_gen_harmonic");
  cudaStreamSynchronize(c->s);
  cudaFree(da);
  return rc;
}

int pc_gen_radial(pc_field* f, const double* tab) {
  field_dep(f);
  if (!f || f->ncomp != 1 || !tab) return fail(PC_E_INVALID, "radial: scalar field and table needed");
  pc_grid* g = f->grid;
  pc_ctx* c = g->ctx;
  double* dt = nullptr;
  TRY(upload_tmp(c, tab, (size_t)g->g.n0g, &dt));
  k_gen_radial<<<node_blocks(c, g->g), kThreads, 0, c->s>>>(g->g, f->base(0), dt);
  c->st.launches++;
  int rc = check_launch("k_gen_radial");
  cudaStreamSynchronize(c->s);
  cudaFree(dt);
  return rc;
}
