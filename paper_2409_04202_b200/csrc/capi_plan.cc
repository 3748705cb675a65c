// C-ABI entry points of the planning core (host only): GenModel fit / closed forms,
// GenTree plans, prediction.  See include/gentree_ar.h for the contract of each call.
#include <cstring>
#include <exception>
#include <new>

#include "../../include/gentree_ar.h"
#include "internal.hpp"

namespace gtar {
static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }
static std::atomic<uint64_t> g_uid{1};
uint64_t next_plan_uid() { return g_uid.fetch_add(1); }
}  // namespace gtar

using namespace gtar;

#define AR_TRY(...)                                   \
  try {                                                \
    __VA_ARGS__                                        \
  } catch (const InvalidArg &e) {                      \
    set_error(e.what());                               \
    return AR_EINVAL;                                  \
  } catch (const std::bad_alloc &) {                   \
    set_error("out of host memory");                   \
    return AR_ESYS;                                    \
  } catch (const std::exception &e) {                  \
    set_error(std::string("internal error: ") + e.what()); \
    return AR_ESYS;                                    \
  }

static Params to_params(const gm_params *p) {
  Params q;
  q.alpha = p->alpha;
  q.beta = p->beta;
  q.gamma = p->gamma;
  q.delta = p->delta;
  q.epsilon = p->epsilon;
  q.w_t = p->w_t;
  q.has_combined = p->has_combined != 0;
  q.combined = p->combined;
  return q;
}

static void check_params(const gm_params *p) {
  if (!(p->alpha >= 0 && p->beta >= 0 && p->gamma >= 0 && p->delta >= 0 && p->epsilon >= 0) || p->w_t < 1 ||
      (p->has_combined && !(p->combined >= 0)))
    throw InvalidArg("GenModel parameters must be non-negative and w_t >= 1");
}

static void fill(gm_breakdown *o, const Breakdown &b) {
  o->latency = b.latency;
  o->bandwidth = b.bandwidth;
  o->compute = b.compute;
  o->memory = b.memory;
  o->incast = b.incast;
  o->total = b.total;
}

extern "C" {

const char *ar_last_error(void) { return g_err.c_str(); }
const char *ar_version(void) { return "gentree_ar 0.1 (sm_100a)"; }

int genmodel_fit(const gm_measurement *rows, size_t n_rows, int32_t wt_min, int32_t wt_max,
                 double link_bytes_per_s, gm_params *out, double *sse) {
  AR_TRY({
    if (!rows || !out) throw InvalidArg("null argument");
    std::vector<Measurement> m;
    for (size_t i = 0; i < n_rows; i++) {
      if (rows[i].n < 2 || rows[i].bytes < 1 || !(rows[i].seconds > 0)) throw InvalidArg("bad measurement row");
      m.push_back({rows[i].n, (double)rows[i].bytes, rows[i].seconds});
    }
    FitResult f = fit_params(m, wt_min, wt_max);
    gm_params o{};
    o.alpha = f.alpha;
    o.delta = f.delta;
    o.epsilon = f.epsilon;
    o.w_t = f.w_t;
    o.combined = f.combined;
    if (link_bytes_per_s > 0) {
      o.beta = 1.0 / link_bytes_per_s;
      o.gamma = f.combined - 2.0 * o.beta;
      if (o.gamma < 0) throw InvalidArg("k < 2*beta: inconsistent inputs (split_combined)");
      o.has_combined = 0;
    } else {
      o.has_combined = 1;
    }
    *out = o;
    if (sse) *sse = f.sse;
    return AR_OK;
  })
}

int genmodel_fit_nvls(const gm_measurement *rows, size_t n_rows, gm_params *out, double *sse) {
  return genmodel_fit_row("nvls", rows, n_rows, out, sse);
}

int genmodel_fit_row(const char *kind, const gm_measurement *rows, size_t n_rows, gm_params *out, double *sse) {
  AR_TRY({
    if (!kind || !rows || !out) throw InvalidArg("null argument");
    const std::string k(kind);
    if (k != "nvls" && k != "oneshot" && k != "ll128")
      throw InvalidArg("genmodel_fit_row: kind must be nvls, oneshot or ll128");
    std::vector<Measurement> m;
    for (size_t i = 0; i < n_rows; i++) {
      if (rows[i].n < 2 || rows[i].bytes < 1 || !(rows[i].seconds > 0)) throw InvalidArg("bad measurement row");
      m.push_back({rows[i].n, (double)rows[i].bytes, rows[i].seconds});
    }
    NvlsFit f = fit_row(k, m);
    gm_params o{};
    o.alpha = f.alpha;
    o.beta = f.beta;
    o.w_t = 1;
    *out = o;
    if (sse) *sse = f.sse;
    return AR_OK;
  })
}

int genmodel_choose_nvls(const gt_plan *plan, const gm_params *plan_params, const gm_params *nvls_params,
                         int32_t *use_nvls, double *t_plan, double *t_nvls) {
  AR_TRY({
    if (!plan || !plan_params || !nvls_params || !use_nvls) throw InvalidArg("null argument");
    check_params(plan_params);
    check_params(nvls_params);
    gm_breakdown bp{};
    if (genmodel_predict_executed(plan, plan_params, &bp) != AR_OK) return AR_EINVAL;
    const int64_t S = plan->plan.count * (int64_t)plan->esize;
    Breakdown bn = closed_form_f64("nvls", plan->plan.n, S, to_params(nvls_params), {});
    *use_nvls = bn.total < bp.total ? 1 : 0;   // ties keep the plan (bit-reproducible order)
    if (t_plan) *t_plan = bp.total;
    if (t_nvls) *t_nvls = bn.total;
    return AR_OK;
  })
}

int gt_plan_simulate(const gt_plan *plan, const char *topology_json, const gm_params *params, gm_breakdown *out,
                     double *step_times, size_t cap, size_t *n_steps) {
  AR_TRY({
    if (!plan || !out) throw InvalidArg("null argument");
    Params p;
    if (params) {
      check_params(params);
      p = to_params(params);
    }
    Topology t = topology_json ? parse_topology(topology_json) : plan->topo;
    if (topology_json && (int)t.servers.size() != plan->plan.n)
      throw InvalidArg("topology and plan have different numbers of ranks");
    if (t.nodes.empty()) {   // plan built from JSON: a single switch with uniform links
      if (!params) throw InvalidArg("a plan without a topology needs explicit params");
      std::string doc = "{\"nodes\":[{\"id\":\"sw\",\"kind\":\"switch\",\"parent\":null,\"uplink\":null}";
      for (int i = 0; i < plan->plan.n; i++)
        doc += ",{\"id\":\"s" + std::to_string(i) +
               "\",\"kind\":\"server\",\"parent\":\"sw\",\"uplink\":{\"alpha\":0,\"beta\":1,\"epsilon\":0,\"w_t\":1},"
               "\"compute\":{\"gamma\":0,\"delta\":0}}";
      doc += "]}";
      t = parse_topology(doc);
    }
    SimResult r = simulate_flows(t, plan->plan, plan->esize, params ? &p : nullptr);
    fill(out, r.b);
    if (n_steps) *n_steps = r.steps.size();
    if (step_times)
      for (size_t i = 0; i < r.steps.size() && i < cap; i++) step_times[i] = r.steps[i];
    return AR_OK;
  })
}

int genmodel_closed_form(const char *kind, int32_t n, uint64_t bytes, const gm_params *params, gm_breakdown *out) {
  AR_TRY({
    if (!kind || !params || !out) throw InvalidArg("null argument");
    check_params(params);
    std::string k(kind);
    std::string name = k;
    std::vector<int> f;
    if (k.rfind("hcps:", 0) == 0) {
      name = "hcps";
      size_t p = 5;
      while (p <= k.size()) {
        size_t q = k.find(',', p);
        if (q == std::string::npos) q = k.size();
        std::string tok = k.substr(p, q - p);
        char *end = nullptr;
        long v = std::strtol(tok.c_str(), &end, 10);
        if (tok.empty() || *end) throw InvalidArg("bad hcps spec");
        f.push_back((int)v);
        p = q + 1;
      }
    }
    fill(out, closed_form_f64(name, n, (int64_t)bytes, to_params(params), f));
    return AR_OK;
  })
}

static int make_plan(const Topology &t, uint64_t count, int32_t dtype, const gm_params *params,
                     const char *force_kind, gt_plan **out) {
  if (!out) throw InvalidArg("null out");
  if (dtype != AR_F32 && dtype != AR_BF16) throw InvalidArg("unknown dtype");
  if (count < 1) throw InvalidArg("count must be >= 1");
  if (count > (uint64_t)1 << 40) throw InvalidArg("count too large");
  Params p;
  if (params) {
    check_params(params);
    p = to_params(params);
  }
  std::string force = force_kind ? force_kind : "";
  const bool nvls = force == "nvls";
  if (nvls) {
    // NVLS plan kind: the single-switch CPS data movement with the
    // reduce in the NVSwitch.  fp32 only: the switch returns the correctly rounded fp32 sum
    // (reading NV2, measured), which has a plain definition to check against; its bf16
    // rounding is not round-to-nearest-even, so bf16 stays on the plan-order kinds.
    if (dtype != AR_F32) throw InvalidArg("NVLS plans are fp32 only (reading NV2: the switch's bf16 rounding is not RNE)");
    int switches = 0;
    for (auto &nd : t.nodes) switches += nd.server ? 0 : 1;
    if (switches != 1) throw InvalidArg("NVLS plans need a single-switch topology (one NVSwitch domain)");
    force = "cps";
  }
  PlanResult r = gentree(t, (int64_t)count, esize_of(dtype), params ? &p : nullptr, force);
  if (nvls) {
    r.plan.switch_reduce = true;
    for (auto &rep : r.reports) rep.chosen = "nvls";
  }
  gt_plan *g = new gt_plan();
  g->plan = std::move(r.plan);
  g->reports = std::move(r.reports);
  g->topo = t;
  g->topo_params = params == nullptr;
  g->dtype = dtype;
  g->esize = esize_of(dtype);
  g->json = plan_to_json(g->plan, dtype_name(dtype));
  g->report = report_to_json(g->reports);
  g->uid = next_plan_uid();
  *out = g;
  return AR_OK;
}

int gentree_plan(const char *topology_json, uint64_t count, int32_t dtype, const gm_params *params,
                 const char *force_kind, gt_plan **out) {
  AR_TRY({
    if (!topology_json) throw InvalidArg("null topology");
    Topology t = parse_topology(topology_json);
    return make_plan(t, count, dtype, params, force_kind, out);
  })
}

int gentree_plan_nvls(const char *topology_json, uint64_t count, int32_t dtype, const gm_params *params,
                      const gm_params *nvls_params, const gm_params *oneshot_params, uint64_t oneshot_max_bytes,
                      const gm_params *ll128_params, uint64_t ll128_min_bytes, uint64_t ll128_max_bytes,
                      gt_plan **out) {
  AR_TRY({
    if (!topology_json || !nvls_params || !params || !out) throw InvalidArg("null argument");
    check_params(nvls_params);
    if (oneshot_params) check_params(oneshot_params);
    if (ll128_params) check_params(ll128_params);
    Topology t = parse_topology(topology_json);
    gt_plan *g = nullptr;
    int rc = make_plan(t, count, dtype, params, nullptr, &g);
    if (rc != AR_OK) return rc;
    int switches = 0;
    for (auto &nd : t.nodes) switches += nd.server ? 0 : 1;
    if (dtype == AR_F32 && switches == 1) {
      int32_t use = 0;
      double tp = 0, tn = 0;
      rc = genmodel_choose_nvls(g, params, nvls_params, &use, &tp, &tn);
      if (rc != AR_OK) {
        delete g;
        return rc;
      }
      const int64_t S = (int64_t)count * esize_of(dtype);
      const bool eligible = !oneshot_order(g->plan).empty();
      const int n = g->plan.n;
      const bool ll128_ok = eligible && n <= 8 && (uint64_t)S >= 8ull * n &&
                            (uint64_t)S > std::min(ll128_min_bytes, oneshot_max_bytes) && (uint64_t)S <= ll128_max_bytes;
      if (ll128_params && ll128_ok) {
        // the executor runs this plan through its LL128 two-shot path (above the LL128 floor):
        // compare that row instead
        tp = closed_form_f64("ll128", n, S, to_params(ll128_params), {}).total;
        use = tn < tp ? 1 : 0;
      } else if (oneshot_params && (uint64_t)S <= oneshot_max_bytes && eligible) {
        // ... or through its one-shot path
        tp = closed_form_f64("oneshot", n, S, to_params(oneshot_params), {}).total;
        use = tn < tp ? 1 : 0;
      }
      if (use) {
        delete g;
        g = nullptr;
        rc = make_plan(t, count, dtype, params, "nvls", &g);
        if (rc != AR_OK) return rc;
      }
    }
    *out = g;
    return AR_OK;
  })
}

int gentree_plan_single_switch(int32_t world, uint64_t count, int32_t dtype, const gm_params *params,
                               const char *force_kind, gt_plan **out) {
  AR_TRY({
    if (!params) throw InvalidArg("params required");
    if (world < 2 || world > 4096) throw InvalidArg("world must be >= 2");
    std::string doc = "{\"nodes\":[{\"id\":\"sw\",\"kind\":\"switch\",\"parent\":null,\"uplink\":null}";
    for (int i = 0; i < world; i++)
      doc += ",{\"id\":\"s" + std::to_string(i) +
             "\",\"kind\":\"server\",\"parent\":\"sw\",\"uplink\":{\"alpha\":0,\"beta\":1,\"epsilon\":0,\"w_t\":1},"
             "\"compute\":{\"gamma\":0,\"delta\":0}}";
    doc += "]}";
    Topology t = parse_topology(doc);
    return make_plan(t, count, dtype, params, force_kind, out);
  })
}

static int copy_out(const std::string &s, char *buf, size_t cap, size_t *needed) {
  if (needed) *needed = s.size() + 1;
  if (!buf || cap < s.size() + 1) {
    set_error("buffer too small");
    return AR_EINVAL;
  }
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return AR_OK;
}

int gt_plan_to_json(const gt_plan *plan, char *buf, size_t cap, size_t *needed) {
  if (!plan) { set_error("null plan"); return AR_EINVAL; }
  return copy_out(plan->json, buf, cap, needed);
}

int gt_plan_report_json(const gt_plan *plan, char *buf, size_t cap, size_t *needed) {
  if (!plan) { set_error("null plan"); return AR_EINVAL; }
  return copy_out(plan->report, buf, cap, needed);
}

int gt_plan_info(const gt_plan *plan, int32_t *n_ranks, int32_t *n_steps, uint64_t *count, int32_t *dtype) {
  if (!plan) { set_error("null plan"); return AR_EINVAL; }
  if (n_ranks) *n_ranks = plan->plan.n;
  if (n_steps) *n_steps = (int32_t)plan->plan.steps.size();
  if (count) *count = (uint64_t)plan->plan.count;
  if (dtype) *dtype = plan->dtype;
  return AR_OK;
}

int genmodel_predict(const gt_plan *plan, const gm_params *params, gm_breakdown *out) {
  AR_TRY({
    if (!plan || !out) throw InvalidArg("null argument");
    if (plan->plan.switch_reduce) {   // NVLS: the NV1 row (no plan-order steps)
      if (!params) throw InvalidArg("an NVLS plan is predicted with explicit (NVLS-row) params");
      check_params(params);
      fill(out, closed_form_f64("nvls", plan->plan.n, plan->plan.count * (int64_t)plan->esize, to_params(params), {}));
      return AR_OK;
    }
    auto co = step_coeffs(plan->plan, plan->esize);
    std::vector<StepParams> sp;
    if (params) {
      check_params(params);
      sp = uniform_step_params(to_params(params), co.size());
    } else {
      if (!plan->topo_params) throw InvalidArg("plan was built with explicit params; pass params");
      sp = topo_step_params(plan->topo, plan->plan);
    }
    fill(out, predict_f64(co, sp));
    return AR_OK;
  })
}

void gt_plan_free(gt_plan *plan) { delete plan; }

int gt_plan_from_json(const char *plan_json, gt_plan **out, int32_t *is_allreduce) {
  AR_TRY({
    if (!plan_json || !out) throw InvalidArg("null argument");
    std::string dtype;
    bool ar = false;
    Plan p = plan_from_json(plan_json, dtype, ar);
    gt_plan *g = new gt_plan();
    g->plan = std::move(p);
    g->topo_params = false;
    g->dtype = dtype == "f32" ? AR_F32 : AR_BF16;
    g->esize = esize_of(g->dtype);
    g->json = plan_to_json(g->plan, dtype.c_str());
    g->report = "[]";
    g->uid = next_plan_uid();
    g->is_allreduce = ar;
    if (is_allreduce) *is_allreduce = ar ? 1 : 0;
    *out = g;
    return AR_OK;
  })
}

}  // extern "C"
