// api.cpp — the C ABI (include/sc_b200.h).  Marshalling and validation only; every arithmetic
// step of the path runs in kernels.cu.
#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "sc_internal.h"

struct sc_plan_s {
  sc::Plan P;
};

namespace {
thread_local std::string g_last_error;

sc_status fail(sc_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
}  // namespace

extern "C" {

void sc_options_default(sc_options* opt) {
  if (!opt) return;
  std::memset(opt, 0, sizeof(*opt));
  opt->precision = 64;
  opt->skip = SC_SKIP_EXACT;
  opt->tile_cols = 0;
  opt->panel_cols = 0;
  opt->n_lambda_global = 0;
  opt->device = 0;
}

sc_status sc_plan_create(const sc_subdomain_desc* sd, int32_t nsub, const sc_options* opt, sc_plan_t* out) {
  if (!out || !opt) return fail(SC_ERR_INVALID_ARG, "sc_plan_create: NULL opt or out");
  *out = nullptr;
  sc_plan_s* h = new (std::nothrow) sc_plan_s();
  if (!h) return fail(SC_ERR_OOM, "host allocation failed");
  std::string err;
  sc_status st;
  try {
    st = sc::build_plan(sd, nsub, *opt, h->P, err);
    if (st == SC_OK && opt->device >= 0) st = sc::upload_plan(h->P, err);
  } catch (const std::bad_alloc&) {
    st = SC_ERR_OOM;
    err = "host allocation failed";
  } catch (...) {
    st = SC_ERR_INVALID_ARG;
    err = "unexpected exception in sc_plan_create";
  }
  if (st != SC_OK) {
    sc::free_plan_device(h->P);
    delete h;
    return fail(st, err);
  }
  *out = h;
  g_last_error.clear();
  return SC_OK;
}

sc_status sc_assemble_batch(sc_plan_t p, const void* const* L_values, void* stream) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  if (!L_values && p->P.nsub > 0) return fail(SC_ERR_INVALID_ARG, "NULL L_values");
  std::string err;
  sc_status st = sc::launch_assemble(p->P, L_values, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_assemble_batch_host(sc_plan_t p, const void* const* L_values_host, void* stream) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  if (!L_values_host && p->P.nsub > 0) return fail(SC_ERR_INVALID_ARG, "NULL L_values_host");
  std::string err;
  sc_status st = sc::assemble_host_pipelined(p->P, L_values_host, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_apply(sc_plan_t p, const double* lambda, double* q, void* stream) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  if ((!lambda || !q) && p->P.n_lambda > 0) return fail(SC_ERR_INVALID_ARG, "NULL lambda or q");
  std::string err;
  sc_status st = sc::launch_apply(p->P, lambda, q, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_prepare_factor(sc_plan_t p, const void* const* L_values, void* stream) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  if (!L_values && p->P.nsub > 0) return fail(SC_ERR_INVALID_ARG, "NULL L_values");
  std::string err;
  sc_status st = sc::launch_prepare(p->P, L_values, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_apply_implicit(sc_plan_t p, const double* lambda, double* q, void* stream) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  if ((!lambda || !q) && p->P.n_lambda > 0) return fail(SC_ERR_INVALID_ARG, "NULL lambda or q");
  std::string err;
  sc_status st = sc::launch_apply_implicit(p->P, lambda, q, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_factor_attach(sc_plan_t p, const sc_K_pattern* K, int32_t nsub) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!K && nsub > 0) return fail(SC_ERR_INVALID_ARG, "NULL K");
  std::string err;
  sc_status st;
  try {
    if (p->P.fac.ready) p->P.stats.device_bytes -= 8.0 * (double)(p->P.fac.W_doubles + p->P.fac.sub_x_base.back());
    sc::free_factor_device(p->P);
    p->P.fac = sc::FactorPlan();
    st = sc::build_factor_plan(p->P, K, nsub, err);
    if (st == SC_OK && p->P.on_device) st = sc::upload_factor_plan(p->P, err);  // host-only: symbolic + stats
  } catch (const std::bad_alloc&) {
    st = SC_ERR_OOM;
    err = "host allocation failed";
  }
  if (st != SC_OK) {
    sc::free_factor_device(p->P);
    p->P.fac = sc::FactorPlan();
    return fail(st, err);
  }
  const sc::FactorPlan& F = p->P.fac;
  sc_stats& S = p->P.stats;
  S.flops_factor_useful = F.flops_useful;
  S.flops_factor_executed = F.flops;
  S.bytes_K_values = F.bytes_K;
  S.factor_tasks = F.task_chunk.empty() ? 0 : F.task_chunk[0];
  S.bytes_factor_W = 8.0 * (double)F.W_doubles;
  S.factor_panels = 0;
  S.factor_max_level = 0;
  for (int32_t i = 0; i < p->P.nsub; i++) {
    const sc::FactorClass& fc = F.classes[(size_t)p->P.sub_cls[(size_t)i]];
    S.factor_panels += (int64_t)fc.panels.size();
    S.factor_max_level = std::max(S.factor_max_level, fc.max_level);
  }
  if (p->P.on_device) S.device_bytes += 8.0 * (double)(F.W_doubles + F.sub_x_base.back());
  return SC_OK;
}

sc_status sc_factorize_batch(sc_plan_t p, const void* const* K_values, void* const* L_values, void* stream) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.fac.ready || !p->P.fac.has_K) return fail(SC_ERR_STATE, "no factorization plan (sc_factor_attach)");
  if ((!K_values || !L_values) && p->P.nsub > 0) return fail(SC_ERR_INVALID_ARG, "NULL K_values or L_values");
  std::string err;
  sc_status st = sc::launch_factorize(p->P, K_values, L_values, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_factorize_assemble_host(sc_plan_t p, const void* const* K_values_host, void* stream) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.fac.ready || !p->P.fac.has_K) return fail(SC_ERR_STATE, "no factorization plan (sc_factor_attach)");
  if (!K_values_host && p->P.nsub > 0) return fail(SC_ERR_INVALID_ARG, "NULL K_values_host");
  std::string err;
  sc_status st = sc::factorize_assemble_host(p->P, K_values_host, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_pcpg(sc_plan_t p, const double* d, const double* e, double* lambda, const sc_coarse* coarse,
                  const sc_pcpg_opts* opts, sc_allreduce_fn allreduce, void* ctx, sc_pcpg_result* res, void* stream) {
  if (!p || !opts) return fail(SC_ERR_INVALID_ARG, "NULL plan or opts");
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  if (p->P.n_lambda > 0 && (!d || !lambda)) return fail(SC_ERR_INVALID_ARG, "NULL d or lambda");
  if (coarse && coarse->nc > 0 &&
      ((!coarse->k || !coarse->off || !coarse->Rt || !coarse->GtG_inv) && p->P.nsub > 0))
    return fail(SC_ERR_INVALID_ARG, "incomplete sc_coarse");
  if (coarse && coarse->nc > 0 && !e) return fail(SC_ERR_INVALID_ARG, "NULL e");
  if (coarse && coarse->nc > 0)
    for (int32_t i = 0; i < p->P.nsub; i++)
      if (coarse->k[i] < 0 || coarse->off[i] < 0 || coarse->off[i] + coarse->k[i] > coarse->nc)
        return fail(SC_ERR_INVALID_ARG, "sc_coarse: subdomain columns outside [0, nc)");
  if (!(opts->rtol >= 0) || opts->max_it < 0) return fail(SC_ERR_INVALID_ARG, "bad rtol / max_it");
  std::string err;
  sc_status st = sc::pcpg_solve(p->P, d, e, lambda, coarse, *opts, allreduce, ctx, res, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_check(sc_plan_t p) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.on_device) return SC_OK;
  std::string err;
  sc_status st = sc::device_check(p->P, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_get_F(sc_plan_t p, int32_t i, double* F, int64_t ld) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  if (i < 0 || i >= p->P.nsub) return fail(SC_ERR_INVALID_ARG, "subdomain index out of range");
  const sc::ClassPlan& C = p->P.classes[(size_t)p->P.sub_cls[(size_t)i]];
  const int64_t m = C.m;
  if (m == 0) return SC_OK;
  if (!F || ld < m) return fail(SC_ERR_INVALID_ARG, "NULL F or ld < m");
  std::string err;
  std::vector<double> Fl;
  sc_status st = sc::copy_F_lower(p->P, i, Fl, err);
  if (st != SC_OK) return fail(st, err);
  // F(sigma(a), sigma(b)) = F'(max(a,b), min(a,b))  (permute back; symmetrise)
  for (int64_t b = 0; b < m; b++)
    for (int64_t a = 0; a < m; a++) {
      const int64_t hi = std::max(a, b), lo = std::min(a, b);
      F[(int64_t)C.sigma[(size_t)b] * ld + C.sigma[(size_t)a]] = Fl[(size_t)sc::f_index((int)hi, (int)lo)];
    }
  return SC_OK;
}

sc_status sc_get_F_device(sc_plan_t p, int32_t i, double* F, int64_t ld, void* stream) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  if (i < 0 || i >= p->P.nsub) return fail(SC_ERR_INVALID_ARG, "subdomain index out of range");
  const int64_t m = p->P.sub_m[(size_t)i];
  if (m == 0) return SC_OK;
  if (!F || ld < m) return fail(SC_ERR_INVALID_ARG, "NULL F or ld < m");
  std::string err;
  sc_status st = sc::export_F_device(p->P, i, F, ld, stream, err);
  return st == SC_OK ? SC_OK : fail(st, err);
}

sc_status sc_get_X(sc_plan_t p, int32_t i, double* X, int32_t* sigma) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (i < 0 || i >= p->P.nsub) return fail(SC_ERR_INVALID_ARG, "subdomain index out of range");
  const sc::ClassPlan& C = p->P.classes[(size_t)p->P.sub_cls[(size_t)i]];
  if (sigma) std::copy(C.sigma.begin(), C.sigma.end(), sigma);
  if (!X) return SC_OK;
  if (!p->P.on_device) return fail(SC_ERR_STATE, "host-only plan (device < 0)");
  std::string err;
  std::vector<double> strips;
  sc_status st = sc::copy_X_strips(p->P, i, strips, err);
  if (st != SC_OK) return fail(st, err);
  const int64_t n = C.n;
  const int32_t cls = p->P.sub_cls[(size_t)i];
  const int32_t panel0 = p->P.cls_panel_begin[(size_t)cls];
  const int32_t greach0 = C.groups.empty() ? 0 : C.groups[0].reach_begin;  // globalised indices
  std::fill(X, X + n * (int64_t)C.m, 0.0);
  for (const sc::Group& G : C.groups)
    for (int32_t q = G.reach_begin; q < G.reach_end; q++) {
      const sc::Reach& R = C.greach[(size_t)(q - greach0)];
      const sc::Panel& pn = C.panels[(size_t)(R.panel - panel0)];
      for (int32_t r = 0; r < pn.kw; r++)
        for (int32_t j = 0; j < G.width; j++)
          X[(int64_t)(G.col0 + j) * n + pn.a + r] = strips[(size_t)(G.x_off + (int64_t)(R.off + r) * p->P.G + j)];
    }
  return SC_OK;
}

sc_status sc_plan_strip_rows(sc_plan_t p, int32_t i, int32_t a, int32_t* rows, int32_t* nrows) {
  if (!p || !rows || !nrows) return fail(SC_ERR_INVALID_ARG, "NULL argument");
  if (i < 0 || i >= p->P.nsub) return fail(SC_ERR_INVALID_ARG, "subdomain index out of range");
  const sc::ClassPlan& C = p->P.classes[(size_t)p->P.sub_cls[(size_t)i]];
  if (a < 0 || a >= C.m) return fail(SC_ERR_INVALID_ARG, "column out of range");
  const int32_t panel0 = p->P.cls_panel_begin[(size_t)p->P.sub_cls[(size_t)i]];
  const int32_t step0 = C.tiles[0].step_begin;  // globalised indices
  const sc::Tile& t = C.tiles[(size_t)(a / p->P.T)];
  int32_t k = 0;
  for (int32_t s = t.step_begin; s < t.step_end; s++) {
    const sc::Panel& pn = C.panels[(size_t)(C.steps[(size_t)(s - step0)].panel - panel0)];
    for (int32_t r = 0; r < pn.kw; r++) rows[k++] = pn.a + r;
  }
  *nrows = k;
  return SC_OK;
}

sc_status sc_plan_stats(sc_plan_t p, sc_stats* out) {
  if (!p || !out) return fail(SC_ERR_INVALID_ARG, "NULL argument");
  *out = p->P.stats;
  return SC_OK;
}

sc_status sc_plan_subdomain_costs(sc_plan_t p, double* costs) {
  if (!p || (!costs && p->P.nsub > 0)) return fail(SC_ERR_INVALID_ARG, "NULL argument");
  for (int32_t i = 0; i < p->P.nsub; i++) {
    const sc::ClassPlan& C = p->P.classes[(size_t)p->P.sub_cls[(size_t)i]];
    costs[i] = C.fl_prep_exec + C.fl_trsm_exec + C.fl_syrk_exec;
  }
  return SC_OK;
}

sc_status sc_set_timing_events(sc_plan_t p, void* const* events, int32_t n) {
  if (!p) return fail(SC_ERR_INVALID_ARG, "NULL plan");
  if (!(n == 0 || (n == 4 && events))) return fail(SC_ERR_INVALID_ARG, "n must be 0 or 4 (with events)");
  for (int k = 0; k < 4; k++) p->P.tev[k] = n ? events[k] : nullptr;
  return SC_OK;
}

int32_t sc_launches_per_assemble(sc_plan_t p) {
  if (!p) return 0;
  int small = 0;
  for (int b = 0; b < 3; b++) small += p->P.small_begin[b + 1] > p->P.small_begin[b] ? 1 : 0;
  if (p->P.warp_trsm) small = 0;
  return (p->P.prep_tasks.empty() || p->P.warp_trsm ? 0 : 1) + small +
         (p->P.trsm_tasks.empty() ? 0 : 1) + (p->P.syrk_tasks.empty() ? 0 : 1);
}

int32_t sc_launches_per_apply_implicit(sc_plan_t p) {
  if (!p) return 0;
  return (p->P.nsub > 0 ? 1 : 0) + (p->P.n_lambda > 0 ? 1 : 0);
}

int32_t sc_launches_per_apply(sc_plan_t p) {
  if (!p) return 0;
  return (p->P.apply_tasks.empty() ? 0 : 1) + (p->P.n_lambda > 0 ? 1 : 0);
}

void sc_plan_destroy(sc_plan_t p) {
  if (!p) return;
  sc::free_plan_device(p->P);
  delete p;
}

const char* sc_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
