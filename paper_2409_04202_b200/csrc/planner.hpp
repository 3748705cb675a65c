// Planning core of the C-ABI library: topology, plans, GenModel, GenTree, fit.
// Written from PAPER.md (arXiv 2409.04202) — citations "P:n" are PAPER.md lines,
// "S:n" SPEC.md lines; readings Qn are the register in DESIGN.md.
// Host-only C++17; compiled with -ffp-contract=off so every double expression rounds
// exactly as written (the fixed evaluation order of DESIGN.md "cost evaluation order").
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace gtar {

struct InvalidArg : std::runtime_error {   // -> AR_EINVAL
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ topology
struct Uplink {
  double alpha = 0, beta = 0, epsilon = 0;   // seconds, seconds per float
  int w_t = 1;
};
struct Compute {
  double gamma = 0, delta = 0;               // seconds per float
};
struct Node {
  std::string id;
  bool server = false;
  int parent = -1;                           // index, -1 for the root
  bool has_uplink = false, has_compute = false;
  Uplink up;
  Compute comp;
  std::vector<int> children;                 // document order
  int rank = -1;                             // servers only
};
struct Topology {
  std::vector<Node> nodes;                   // document order
  int root = -1;
  std::vector<int> servers;                  // rank -> node index (DFS pre-order)
  void servers_under(int n, std::vector<int> &out) const;   // ranks
  void subtree(int n, std::vector<int> &out) const;
  std::vector<int> path_links(int a, int b) const;          // node indices
  double convergence_ratio_f64(int sw, int child) const;
  int rearrangement_subset_size(int sw, int child, int ni) const;   // exact ceil(n_i / r), reading Q15
};
Topology parse_topology(const std::string &text);           // throws InvalidArg

// ------------------------------------------------------------------ plans
struct Reduce {
  int server, block;
  std::vector<int> inputs;                   // summation order (ascending rank, Q1)
};
struct Transfer {
  int src, dst, block;
  int64_t size;                              // elements
};
struct Step {
  bool ag = false;                           // phase: false = rs, true = ag
  std::string label;
  std::vector<Reduce> reduces;
  std::vector<Transfer> transfers;
};
struct Plan {
  int n = 0;
  int64_t count = 0;
  std::vector<Step> steps;
  // NVLS plan kind (readings NV1/NV2): CPS's data movement with every
  // fan-in-N reduce done inside the NVSwitch — the result is the correctly rounded sum, not
  // a plan-order sum.  Serialised as "switch_reduce": true.
  bool switch_reduce = false;
};

int64_t block_size(int64_t count, int n, int b);
int64_t block_offset(int64_t count, int n, int b);

// ------------------------------------------------------------------ GenModel
struct Params {                              // per byte
  double alpha = 0, beta = 0, gamma = 0, delta = 0, epsilon = 0;
  int w_t = 1;
  bool has_combined = false;
  double combined = 0;
  void effective(double &b, double &g) const {
    if (has_combined) { b = combined * 0.5; g = 0.0; }
    else { b = beta; g = gamma; }
  }
};
struct StepCoeffs { int64_t A, B, C, D; int w; };
struct StepParams { double alpha, beta, epsilon; int w_t; double gamma, delta; };
struct Breakdown { double latency = 0, bandwidth = 0, compute = 0, memory = 0, incast = 0, total = 0; };

std::vector<StepCoeffs> step_coeffs(const Plan &p, int esize);
std::vector<StepParams> topo_step_params(const Topology &t, const Plan &p);
std::vector<StepParams> uniform_step_params(const Params &p, size_t n);
Breakdown predict_f64(const std::vector<StepCoeffs> &c, const std::vector<StepParams> &p);
Breakdown closed_form_f64(const std::string &kind, int c, int64_t S, const Params &p,
                          const std::vector<int> &fanins);
std::vector<std::vector<int>> hcps_factorizations(int n, int max_steps);

// ------------------------------------------------------------------ GenTree
struct SwitchReport {
  std::string sw, chosen;
  std::vector<std::pair<std::string, double>> candidates;
  std::vector<std::string> rearranged;
  double start_time = 0, finish_time = 0;
};
struct PlanResult {
  Plan plan;
  std::vector<SwitchReport> reports;
};
// force: "" = GenTree; "cps" | "ring" | "rhd" | "rb" | "hcps:f0,f1,..".
PlanResult gentree(const Topology &t, int64_t count, int esize, const Params *explicit_params,
                   const std::string &force);
Plan build_plan_natural(const std::string &kind, int n, int64_t count);   // standalone
// Parse the canonical plan JSON (plan_to_json's format).  Checks structure, block indices
// and sizes, and the within-step hazard rule; `allreduce` is set iff the plan also passes
// verify_allreduce (data-movement probes need not).  Throws InvalidArg.
Plan plan_from_json(const std::string &text, std::string &dtype, bool &allreduce);
void verify_allreduce(const Plan &p);                                      // throws InvalidArg
void check_switch_reduce(const Plan &p);                                   // NVLS plans: CPS shape
std::vector<int> oneshot_order(const Plan &p);   // one-shot-eligible plans: the common input order
std::string plan_to_json(const Plan &p, const char *dtype);
std::string report_to_json(const std::vector<SwitchReport> &r);

// ------------------------------------------------------------------ flow simulator (NEXT #2)
struct SimResult {
  Breakdown b;                       // latency, bandwidth (ε = 0), incast, compute, memory, total
  std::vector<double> steps;         // per-step time
};
// params == nullptr: each link's / server's own parameters from the topology (per float / 4)
SimResult simulate_flows(const Topology &t, const Plan &p, int esize, const Params *params);

// ------------------------------------------------------------------ fit
struct Measurement { int n; double s; double t; };
struct FitResult {
  double alpha = 0, combined = 0, delta = 0, epsilon = 0, sse = 0;
  int w_t = 0;
};
FitResult fit_params(const std::vector<Measurement> &rows, int wt_min, int wt_max);
struct NvlsFit { double alpha = 0, beta = 0, sse = 0; };
NvlsFit fit_nvls(const std::vector<Measurement> &rows);   // NVLS row (reading NV1)
NvlsFit fit_row(const std::string &kind, const std::vector<Measurement> &rows);   // (α, β) of a row

}  // namespace gtar
