// Incast-aware flow-level simulation of a plan ("a custom-made
// flow-level network simulator which is aware of the incast problem"; procedure S:382-424 with
// DESIGN.md readings FS1-FS3).  Per step: flows = the step's transfers routed on the tree
// path; α = max over used links (Q16); communication time by progressive filling (max-min
// fair rates, recomputed at each flow completion) with per-directed-link capacity 1/β' and
// β' = β + max(w − w_t, 0)·ε, w = 1 + distinct source ranks of the active flows on the link
// (FS1); compute = max over servers of Σ (k−1)|b|γ + (k+1)|b|δ over its k >= 2 reduces.
// Double precision; ties in the filling within 1e-12 relative.
#include <algorithm>
#include <cmath>

#include "planner.hpp"

namespace gtar {

namespace {

struct LinkP { double alpha, beta, eps; int w_t; };

struct Flow {
  int src;
  double bytes;
  std::vector<int> links;   // directed link ids: node*2 + (0 up, 1 down)
};

// max-min rates of the active flows; rate < 0 means unconstrained (infinite)
void max_min(const std::vector<Flow> &flows, const std::vector<int> &active, const std::vector<LinkP> &lp,
             bool incast, std::vector<double> &rate) {
  std::vector<std::vector<int>> on;
  std::vector<int> ids;   // used link ids
  std::vector<int> slot(lp.size() * 2, -1);
  for (int i : active)
    for (int l : flows[i].links) {
      if (slot[l] < 0) {
        slot[l] = (int)on.size();
        on.emplace_back();
        ids.push_back(l);
      }
      on[slot[l]].push_back(i);
    }
  const size_t L = on.size();
  std::vector<double> resid(L);
  std::vector<char> unconstrained(L, 0);
  for (size_t k = 0; k < L; k++) {
    const LinkP &p = lp[ids[k] / 2];
    std::vector<int> srcs;
    for (int i : on[k]) srcs.push_back(flows[i].src);
    std::sort(srcs.begin(), srcs.end());
    const int w = 1 + (int)(std::unique(srcs.begin(), srcs.end()) - srcs.begin());
    const double bp = p.beta + (incast ? (double)std::max(w - p.w_t, 0) * p.eps : 0.0);
    if (bp == 0.0) unconstrained[k] = 1;
    else resid[k] = 1.0 / bp;
  }
  std::vector<char> frozen(flows.size(), 1);
  for (int i : active) frozen[i] = 0;
  size_t left = active.size();
  std::vector<int> cnt(L);
  while (left > 0) {
    double best = -1;
    for (size_t k = 0; k < L; k++) {
      if (unconstrained[k]) continue;
      int c = 0;
      for (int i : on[k]) c += !frozen[i];
      cnt[k] = c;
      if (c == 0) continue;
      const double share = resid[k] / c;
      if (best < 0 || share < best) best = share;
    }
    if (best < 0) {
      for (int i : active)
        if (!frozen[i]) { rate[i] = -1; frozen[i] = 1; }
      break;
    }
    std::vector<int> fr;
    for (size_t k = 0; k < L; k++) {
      if (unconstrained[k] || cnt[k] == 0) continue;
      if (resid[k] / cnt[k] <= best * (1 + 1e-12))
        for (int i : on[k])
          if (!frozen[i]) fr.push_back(i);
    }
    std::sort(fr.begin(), fr.end());
    fr.erase(std::unique(fr.begin(), fr.end()), fr.end());
    for (int i : fr) {
      rate[i] = best;
      frozen[i] = 1;
      left--;
      for (int l : flows[i].links) {
        const int k = slot[l];
        if (!unconstrained[k]) resid[k] -= best;
      }
    }
  }
}

double comm_time(const std::vector<Flow> &flows, const std::vector<LinkP> &lp, bool incast) {
  std::vector<double> rem(flows.size());
  std::vector<int> active;
  for (size_t i = 0; i < flows.size(); i++) {
    rem[i] = flows[i].bytes;
    if (rem[i] > 0) active.push_back((int)i);
  }
  std::vector<double> rate(flows.size(), 0.0);
  double t = 0;
  while (!active.empty()) {
    max_min(flows, active, lp, incast, rate);
    std::vector<int> next;
    bool any_inf = false;
    for (int i : active)
      if (rate[i] < 0) any_inf = true;
    if (any_inf) {
      for (int i : active)
        if (rate[i] >= 0) next.push_back(i);
      active.swap(next);
      continue;
    }
    double dt = -1;
    for (int i : active) {
      const double d = rem[i] / rate[i];
      if (dt < 0 || d < dt) dt = d;
    }
    t += dt;
    for (int i : active) {
      rem[i] -= rate[i] * dt;
      if (rem[i] > flows[i].bytes * 1e-12) next.push_back(i);
    }
    active.swap(next);
  }
  return t;
}

std::vector<int> route(const Topology &t, int a, int b) {
  std::vector<int> ua{a}, ub{b};
  while (t.nodes[ua.back()].parent >= 0) ua.push_back(t.nodes[ua.back()].parent);
  while (t.nodes[ub.back()].parent >= 0) ub.push_back(t.nodes[ub.back()].parent);
  int lca = -1;
  for (int x : ub)
    if (std::find(ua.begin(), ua.end(), x) != ua.end()) { lca = x; break; }
  std::vector<int> out;
  for (int x : ua) {
    if (x == lca) break;
    out.push_back(x * 2);
  }
  std::vector<int> down;
  for (int x : ub) {
    if (x == lca) break;
    down.push_back(x * 2 + 1);
  }
  out.insert(out.end(), down.rbegin(), down.rend());
  return out;
}

}  // namespace

SimResult simulate_flows(const Topology &t, const Plan &p, int esize, const Params *params) {
  std::vector<LinkP> lp(t.nodes.size(), LinkP{0, 0, 0, 1});
  double ub = 0, ug = 0;
  if (params) params->effective(ub, ug);
  for (size_t i = 0; i < t.nodes.size(); i++) {
    const Node &nd = t.nodes[i];
    if (!nd.has_uplink) continue;
    if (params) lp[i] = {params->alpha, ub, params->epsilon, params->w_t};
    else lp[i] = {nd.up.alpha, nd.up.beta / 4.0, nd.up.epsilon / 4.0, nd.up.w_t};
  }
  const int n = p.n;
  std::vector<double> gam(n), del(n);
  for (int r = 0; r < n; r++) {
    if (params) {
      gam[r] = ug;
      del[r] = params->delta;
    } else {
      gam[r] = t.nodes[t.servers[r]].comp.gamma / 4.0;
      del[r] = t.nodes[t.servers[r]].comp.delta / 4.0;
    }
  }
  SimResult res;
  for (const Step &st : p.steps) {
    std::vector<Flow> flows;
    for (const Transfer &tr : st.transfers) {
      if (tr.size <= 0 || tr.src == tr.dst) continue;
      flows.push_back({tr.src, (double)(tr.size * esize), route(t, t.servers[tr.src], t.servers[tr.dst])});
    }
    double a = 0;
    for (const Flow &f : flows)
      for (int l : f.links) a = std::max(a, lp[l / 2].alpha);
    const double c_full = comm_time(flows, lp, true);
    const double c_bw = comm_time(flows, lp, false);
    std::vector<double> g(n, 0.0), d(n, 0.0);
    for (const Reduce &rd : st.reduces) {
      const int k = (int)rd.inputs.size();
      if (k < 2) continue;
      const double sz = (double)(block_size(p.count, n, rd.block) * esize);
      g[rd.server] += (double)(k - 1) * sz * gam[rd.server];
      d[rd.server] += (double)(k + 1) * sz * del[rd.server];
    }
    int slow = 0;
    for (int r = 1; r < n; r++)
      if (g[r] + d[r] > g[slow] + d[slow]) slow = r;
    const double step = ((a + c_full) + (g[slow] + d[slow]));
    res.steps.push_back(step);
    res.b.latency += a;
    res.b.bandwidth += c_bw;
    res.b.incast += c_full - c_bw;
    res.b.compute += g[slow];
    res.b.memory += d[slow];
    res.b.total += step;
  }
  return res;
}

}  // namespace gtar
