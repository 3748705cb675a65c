// Planning core: topology, plan builders, GenModel, GenTree (Alg. 1 + 2), fit.
// See planner.hpp.  Every double expression here is evaluated in the order written
// (built with -ffp-contract=off); the order is the contract of DESIGN.md
// "cost evaluation order", which the CPU oracle follows independently.
#include "planner.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <numeric>
#include <set>
#include <sstream>
#include <tuple>

#include "json.hpp"

namespace gtar {

// ====================================================================== topology
static double num_of(const Json &v, const char *what) {
  if (v.kind != Json::Number) throw InvalidArg(std::string(what) + " must be a number");
  return v.num;
}

Topology parse_topology(const std::string &text) {
  Json doc;
  try {
    doc = JsonReader(text).parse();
  } catch (const JsonError &e) {
    throw InvalidArg(e.what());
  }
  if (doc.kind != Json::Object || doc.obj.size() != 1 || doc.obj[0].first != "nodes" ||
      doc.obj[0].second.kind != Json::Array)
    throw InvalidArg("top level must be {\"nodes\": [...]}");
  Topology t;
  std::map<std::string, int> idx;
  for (const Json &nd : doc.obj[0].second.arr) {
    if (nd.kind != Json::Object) throw InvalidArg("node must be an object");
    for (auto &kv : nd.obj) {
      const std::string &k = kv.first;
      if (k != "id" && k != "kind" && k != "parent" && k != "uplink" && k != "compute")
        throw InvalidArg("unknown key " + k);
    }
    Node n;
    const Json *id = nd.get("id");
    if (!id || id->kind != Json::String || id->str.empty()) throw InvalidArg("node id must be a non-empty string");
    n.id = id->str;
    if (idx.count(n.id)) throw InvalidArg("duplicate id " + n.id);
    const Json *kind = nd.get("kind");
    if (!kind || kind->kind != Json::String || (kind->str != "switch" && kind->str != "server"))
      throw InvalidArg("bad kind for " + n.id);
    n.server = kind->str == "server";
    const Json *par = nd.get("parent");
    if (par && par->kind != Json::Null && par->kind != Json::String)
      throw InvalidArg("parent must be a string or null");
    const Json *up = nd.get("uplink");
    if (up && up->kind != Json::Null) {
      if (up->kind != Json::Object || up->obj.size() != 4 || !up->get("alpha") || !up->get("beta") ||
          !up->get("epsilon") || !up->get("w_t"))
        throw InvalidArg("uplink of " + n.id + " needs exactly alpha, beta, epsilon, w_t");
      const Json *wt = up->get("w_t");
      if (wt->kind != Json::Number || !wt->is_integer || wt->ival < 1) throw InvalidArg("w_t must be an integer >= 1");
      n.has_uplink = true;
      n.up.alpha = num_of(*up->get("alpha"), "alpha");
      n.up.beta = num_of(*up->get("beta"), "beta");
      n.up.epsilon = num_of(*up->get("epsilon"), "epsilon");
      n.up.w_t = (int)wt->ival;
      if (n.up.alpha < 0 || n.up.beta <= 0 || n.up.epsilon < 0)
        throw InvalidArg("need alpha >= 0, beta > 0, epsilon >= 0");
    }
    const Json *cp = nd.get("compute");
    if (cp && cp->kind != Json::Null) {
      if (cp->kind != Json::Object || cp->obj.size() != 2 || !cp->get("gamma") || !cp->get("delta"))
        throw InvalidArg("compute of " + n.id + " needs exactly gamma, delta");
      n.has_compute = true;
      n.comp.gamma = num_of(*cp->get("gamma"), "gamma");
      n.comp.delta = num_of(*cp->get("delta"), "delta");
      if (n.comp.gamma < 0 || n.comp.delta < 0) throw InvalidArg("need gamma, delta >= 0");
    }
    idx[n.id] = (int)t.nodes.size();
    t.nodes.push_back(n);
  }
  // second pass: parents (by id) — kept as strings until every id is known
  std::vector<std::string> parent_ids;
  {
    const Json &arr = doc.obj[0].second;
    for (const Json &nd : arr.arr) {
      const Json *par = nd.get("parent");
      parent_ids.push_back(par && par->kind == Json::String ? par->str : std::string("\x01"));
    }
  }
  int nroots = 0;
  for (size_t i = 0; i < t.nodes.size(); i++)
    if (parent_ids[i] == "\x01") { nroots++; t.root = (int)i; }
  if (nroots != 1) throw InvalidArg("need exactly one root, found " + std::to_string(nroots));
  for (size_t i = 0; i < t.nodes.size(); i++) {
    Node &n = t.nodes[i];
    if (parent_ids[i] != "\x01") {
      auto it = idx.find(parent_ids[i]);
      if (it == idx.end()) throw InvalidArg("parent of " + n.id + " does not exist");
      n.parent = it->second;
      t.nodes[n.parent].children.push_back((int)i);
      if (!n.has_uplink) throw InvalidArg("non-root " + n.id + " needs an uplink");
    } else if (n.has_uplink) {
      throw InvalidArg("root must not have an uplink");
    }
  }
  std::vector<char> seen(t.nodes.size(), 0);
  std::vector<int> stack{t.root};
  size_t nseen = 0;
  while (!stack.empty()) {
    int x = stack.back();
    stack.pop_back();
    if (seen[x]) throw InvalidArg("cycle");
    seen[x] = 1;
    nseen++;
    for (int c : t.nodes[x].children) stack.push_back(c);
  }
  if (nseen != t.nodes.size()) throw InvalidArg("cycle or disconnected node");
  for (auto &n : t.nodes) {
    if (n.server) {
      if (!n.children.empty()) throw InvalidArg("server " + n.id + " has children");
      if (!n.has_compute) throw InvalidArg("server " + n.id + " needs compute params");
    } else {
      if (n.children.empty()) throw InvalidArg("switch " + n.id + " is a leaf");
      if (n.has_compute) throw InvalidArg("switch " + n.id + " must not have compute params");
    }
  }
  std::function<void(int)> dfs = [&](int x) {
    if (t.nodes[x].server) {
      t.nodes[x].rank = (int)t.servers.size();
      t.servers.push_back(x);
    }
    for (int c : t.nodes[x].children) dfs(c);
  };
  dfs(t.root);
  if (t.servers.size() < 2) throw InvalidArg("fewer than 2 servers");
  return t;
}

void Topology::servers_under(int n, std::vector<int> &out) const {
  if (nodes[n].server) out.push_back(nodes[n].rank);
  for (int c : nodes[n].children) servers_under(c, out);
}

void Topology::subtree(int n, std::vector<int> &out) const {
  out.push_back(n);
  for (int c : nodes[n].children) subtree(c, out);
}

std::vector<int> Topology::path_links(int a, int b) const {
  std::vector<int> ua{a}, ub{b};
  while (nodes[ua.back()].parent >= 0) ua.push_back(nodes[ua.back()].parent);
  while (nodes[ub.back()].parent >= 0) ub.push_back(nodes[ub.back()].parent);
  int lca = -1;
  for (int x : ub)
    if (std::find(ua.begin(), ua.end(), x) != ua.end()) { lca = x; break; }
  std::vector<int> out;
  for (int x : ua) { if (x == lca) break; out.push_back(x); }
  for (int x : ub) { if (x == lca) break; out.push_back(x); }
  return out;
}

// ---- exact rearrangement subset size (reading Q15): the smallest m >= 1 with
// m * r >= n_i, r = beta_i * sum_k 1/beta_k, decided exactly.  Every beta is a double
// M * 2^E (M a 53-bit integer); multiplying m * sum_k M_i 2^(E_i - E_k) / M_k >= n_i through by
// prod_j M_j * 2^t leaves integers only, compared with a small unsigned big-integer type.
namespace {
struct BigU {
  std::vector<uint64_t> d;   // little-endian 64-bit limbs
  explicit BigU(uint64_t v = 0) { d.push_back(v); }
  void trim() { while (d.size() > 1 && d.back() == 0) d.pop_back(); }
  void mul(uint64_t m) {
    unsigned __int128 carry = 0;
    for (auto &x : d) {
      unsigned __int128 p = (unsigned __int128)x * m + carry;
      x = (uint64_t)p;
      carry = p >> 64;
    }
    if (carry) d.push_back((uint64_t)carry);
    trim();
  }
  void shl(int bits) {
    const int w = bits / 64, b = bits % 64;
    if (b) {
      uint64_t carry = 0;
      for (auto &x : d) {
        const uint64_t nx = (x << b) | carry;
        carry = x >> (64 - b);
        x = nx;
      }
      if (carry) d.push_back(carry);
    }
    d.insert(d.begin(), (size_t)w, 0ull);
    trim();
  }
  void add(const BigU &o) {
    if (o.d.size() > d.size()) d.resize(o.d.size(), 0);
    unsigned __int128 carry = 0;
    for (size_t i = 0; i < d.size(); i++) {
      unsigned __int128 s = (unsigned __int128)d[i] + (i < o.d.size() ? o.d[i] : 0) + carry;
      d[i] = (uint64_t)s;
      carry = s >> 64;
    }
    if (carry) d.push_back((uint64_t)carry);
  }
  int cmp(const BigU &o) const {
    if (d.size() != o.d.size()) return d.size() < o.d.size() ? -1 : 1;
    for (size_t i = d.size(); i-- > 0;)
      if (d[i] != o.d[i]) return d[i] < o.d[i] ? -1 : 1;
    return 0;
  }
};
void split_double(double b, uint64_t &m, int &e) {
  int ex = 0;
  const double f = std::frexp(b, &ex);   // b = f * 2^ex, 0.5 <= f < 1
  m = (uint64_t)std::ldexp(f, 53);       // exact: a double has 53 significant bits
  e = ex - 53;
}
}  // namespace

int Topology::rearrangement_subset_size(int sw, int child, int ni) const {
  const auto &ch = nodes[sw].children;
  const int K = (int)ch.size();
  std::vector<uint64_t> M(K);
  std::vector<int> E(K);
  for (int k = 0; k < K; k++) split_double(nodes[ch[k]].up.beta, M[k], E[k]);
  uint64_t Mi;
  int Ei;
  split_double(nodes[child].up.beta, Mi, Ei);
  int smin = 0;
  for (int k = 0; k < K; k++) smin = std::min(smin, Ei - E[k]);
  const int tsh = -smin;   // >= 0: every 2^(s_k + t) is an integer power
  // S = sum_k M_i * prod_{j != k} M_j * 2^(E_i - E_k + t);  R = n_i * prod_j M_j * 2^t
  BigU S(0);
  for (int k = 0; k < K; k++) {
    BigU term(Mi);
    for (int j = 0; j < K; j++)
      if (j != k) term.mul(M[j]);
    term.shl(Ei - E[k] + tsh);
    S.add(term);
  }
  BigU R((uint64_t)ni);
  for (int j = 0; j < K; j++) R.mul(M[j]);
  R.shl(tsh);
  for (int m = 1; m <= ni; m++) {
    BigU lhs = S;
    lhs.mul((uint64_t)m);
    if (lhs.cmp(R) >= 0) return m;
  }
  return ni;
}

double Topology::convergence_ratio_f64(int sw, int child) const {
  double acc = 0.0;
  for (int c : nodes[sw].children) acc = acc + 1.0 / nodes[c].up.beta;
  return nodes[child].up.beta * acc;
}

// ====================================================================== plans
int64_t block_size(int64_t count, int n, int b) { return count / n + (b < count % n ? 1 : 0); }
int64_t block_offset(int64_t count, int n, int b) {
  return (int64_t)b * (count / n) + std::min<int64_t>(b, count % n);
}

static bool is_pow2(int x) { return x >= 1 && (x & (x - 1)) == 0; }
static int ilog2(int x) { int k = 0; while ((1 << (k + 1)) <= x) k++; return k; }
static int ceil_log2(int c) { int k = 0; while ((1 << k) < c) k++; return k; }
static int bitrev(int j, int bits) {
  int r = 0;
  for (int k = 0; k < bits; k++)
    if (j & (1 << k)) r |= 1 << (bits - 1 - k);
  return r;
}

struct NatOp { int part, chunk; std::vector<int> ins; };
using NatStep = std::vector<NatOp>;

// Natural RS over c participants / c chunks; natowner[j] = final holder of chunk j.
// cps P:141, ring P:143 (Q10), rhd P:145 (Q11), hcps P:474/P:478 (Q4), rb P:136.
static std::vector<NatStep> natural_rs(const std::string &kind, int c, const std::vector<int> &f,
                                       std::vector<int> &natowner) {
  if (c < 2) throw InvalidArg("need at least 2 participants");
  std::vector<NatStep> steps;
  natowner.assign(c, 0);
  std::vector<int> all(c);
  std::iota(all.begin(), all.end(), 0);
  if (kind == "cps") {
    NatStep st;
    for (int k = 0; k < c; k++) st.push_back({k, k, all});
    steps.push_back(st);
    for (int j = 0; j < c; j++) natowner[j] = j;
  } else if (kind == "rb") {
    NatStep st;
    for (int j = 0; j < c; j++) st.push_back({0, j, all});
    steps.push_back(st);
  } else if (kind == "ring") {
    for (int j = 0; j < c - 1; j++) {
      NatStep st;
      for (int i = 0; i < c; i++)
        st.push_back({i, ((i - j) % c + c) % c, {((i - 1) % c + c) % c, i}});
      steps.push_back(st);
    }
    for (int k = 0; k < c; k++) natowner[k] = ((k - 2) % c + c) % c;
  } else if (kind == "rhd") {
    if (!is_pow2(c)) throw InvalidArg("natural rhd needs a power-of-two participant count");
    int bits = ilog2(c);
    std::vector<int> lo(c, 0), hi(c, c);
    for (int k = 0; k < bits; k++) {
      int mask = 1 << k;
      NatStep st;
      std::vector<int> nlo = lo, nhi = hi;
      for (int i = 0; i < c; i++) {
        int p = i ^ mask;
        int mid = (lo[i] + hi[i]) / 2;
        if (i & mask) nlo[i] = mid; else nhi[i] = mid;
        for (int j = nlo[i]; j < nhi[i]; j++) st.push_back({i, j, {std::min(i, p), std::max(i, p)}});
      }
      lo = nlo;
      hi = nhi;
      steps.push_back(st);
    }
    for (int j = 0; j < c; j++) natowner[j] = bitrev(j, bits);
  } else if (kind == "hcps") {
    long long prod = 1;
    for (int x : f) {
      if (x < 2) throw InvalidArg("hcps fan-ins must be >= 2");
      prod *= x;
    }
    if (f.empty() || prod != c) throw InvalidArg("hcps fan-ins do not multiply to the group size");
    int m = (int)f.size();
    auto digits = [&](int k) {
      std::vector<int> d(m);
      for (int i = 0; i < m; i++) { d[i] = k % f[i]; k /= f[i]; }
      return d;
    };
    auto place = [&](const std::vector<int> &d) {
      int k = 0, mul = 1;
      for (int i = 0; i < m; i++) { k += d[i] * mul; mul *= f[i]; }
      return k;
    };
    for (int i = 0; i < m; i++) {
      NatStep st;
      for (int k = 0; k < c; k++) {
        std::vector<int> d = digits(k);
        int lo = 0, size = c;
        for (int l = 0; l <= i; l++) { size /= f[l]; lo += d[l] * size; }
        std::vector<int> group;
        for (int x = 0; x < f[i]; x++) {
          std::vector<int> dd = d;
          dd[i] = x;
          group.push_back(place(dd));
        }
        for (int j = lo; j < lo + size; j++) st.push_back({k, j, group});
      }
      steps.push_back(st);
    }
    for (int j = 0; j < c; j++) {
      std::vector<int> d;
      int rem = j, size = c;
      for (int i = 0; i < m; i++) { size /= f[i]; d.push_back(rem / size); rem %= size; }
      natowner[j] = place(d);
    }
  } else {
    throw InvalidArg("unknown kind " + kind);
  }
  return steps;
}

static std::vector<Step> realize(const std::vector<NatStep> &nat,
                                 const std::vector<std::vector<int>> &chunk_blocks,
                                 const std::vector<int> &parts, const std::string &label) {
  std::vector<Step> out;
  for (const NatStep &st : nat) {
    Step s;
    s.label = label;
    for (const NatOp &op : st) {
      int r = parts[op.part];
      std::vector<int> ranks;
      for (int q : op.ins) ranks.push_back(parts[q]);
      std::sort(ranks.begin(), ranks.end());
      for (int b : chunk_blocks[op.chunk]) s.reduces.push_back({r, b, ranks});
    }
    out.push_back(std::move(s));
  }
  return out;
}

static void add_implied_transfers(Step &st, int64_t count, int n) {
  st.transfers.clear();
  for (const Reduce &rd : st.reduces)
    for (int q : rd.inputs)
      if (q != rd.server) st.transfers.push_back({q, rd.server, rd.block, block_size(count, n, rd.block)});
}

static std::vector<Step> reverse_to_allgather(const std::vector<Step> &rs) {
  std::vector<Step> ag;
  for (auto it = rs.rbegin(); it != rs.rend(); ++it) {
    Step s;
    s.ag = true;
    s.label = it->label;
    for (const Transfer &t : it->transfers) s.transfers.push_back({t.dst, t.src, t.block, t.size});
    ag.push_back(std::move(s));
  }
  return ag;
}

static void parse_kind(const std::string &kind, std::string &name, std::vector<int> &f) {
  f.clear();
  if (kind.rfind("hcps:", 0) == 0) {
    name = "hcps";
    std::stringstream ss(kind.substr(5));
    std::string tok;
    while (std::getline(ss, tok, ',')) {
      char *end = nullptr;
      long v = std::strtol(tok.c_str(), &end, 10);
      if (tok.empty() || *end != '\0') throw InvalidArg("bad hcps spec " + kind);
      f.push_back((int)v);
    }
    return;
  }
  if (kind == "cps" || kind == "ring" || kind == "rhd" || kind == "rb") { name = kind; return; }
  throw InvalidArg("unknown kind " + kind);
}

static std::string kind_label(const std::string &name, const std::vector<int> &f) {
  if (name != "hcps") return name;
  std::string s = "hcps[";
  for (size_t i = 0; i < f.size(); i++) s += (i ? "," : "") + std::to_string(f[i]);
  return s + "]";
}

Plan build_plan_natural(const std::string &kind, int n, int64_t count) {
  if (n < 2) throw InvalidArg("fewer than 2 servers");
  if (count < 1) throw InvalidArg("count must be >= 1");
  std::string name;
  std::vector<int> f;
  parse_kind(kind, name, f);
  if (name == "rhd" && !is_pow2(n)) throw InvalidArg("non-power-of-two rhd is oracle-only");
  std::vector<int> natowner;
  auto nat = natural_rs(name, n, f, natowner);
  std::vector<std::vector<int>> chunks(n);
  for (int j = 0; j < n; j++) chunks[j] = {j};
  std::vector<int> parts(n);
  std::iota(parts.begin(), parts.end(), 0);
  auto rs = realize(nat, chunks, parts, kind_label(name, f));
  for (auto &s : rs) add_implied_transfers(s, count, n);
  Plan p;
  p.n = n;
  p.count = count;
  p.steps = rs;
  auto ag = reverse_to_allgather(rs);
  p.steps.insert(p.steps.end(), ag.begin(), ag.end());
  return p;
}

// ---------------------------------------------------------------- verification
void verify_allreduce(const Plan &p) {
  const int n = p.n;
  const int W = (n + 63) / 64;
  std::vector<uint64_t> tags((size_t)n * n * W, 0), nt;
  auto T = [&](std::vector<uint64_t> &v, int r, int b) { return &v[((size_t)r * n + b) * W]; };
  for (int r = 0; r < n; r++)
    for (int b = 0; b < n; b++) T(tags, r, b)[r / 64] |= 1ull << (r % 64);
  for (size_t si = 0; si < p.steps.size(); si++) {
    const Step &st = p.steps[si];
    // hazard check: no (rank, block) written twice or written while read by another op
    std::map<std::pair<int, int>, int> writes;
    std::map<std::pair<int, int>, std::set<int>> reads;
    if (!st.ag) {
      for (size_t i = 0; i < st.reduces.size(); i++) {
        auto w = std::make_pair(st.reduces[i].server, st.reduces[i].block);
        if (writes.count(w)) throw InvalidArg("plan hazard: block written twice in step " + std::to_string(si));
        writes[w] = (int)i;
        for (int q : st.reduces[i].inputs) reads[{q, st.reduces[i].block}].insert((int)i);
      }
    } else {
      for (size_t i = 0; i < st.transfers.size(); i++) {
        auto w = std::make_pair(st.transfers[i].dst, st.transfers[i].block);
        if (writes.count(w)) throw InvalidArg("plan hazard: block written twice in step " + std::to_string(si));
        writes[w] = (int)i;
        reads[{st.transfers[i].src, st.transfers[i].block}].insert((int)i);
      }
    }
    for (auto &kv : writes) {
      auto it = reads.find(kv.first);
      if (it == reads.end()) continue;
      for (int o : it->second)
        if (o != kv.second) throw InvalidArg("plan hazard: read/write conflict in step " + std::to_string(si));
    }
    nt = tags;
    if (!st.ag) {
      for (const Reduce &rd : st.reduces) {
        uint64_t *dst = T(nt, rd.server, rd.block);
        std::vector<uint64_t> acc(W, 0);
        for (int q : rd.inputs) {
          const uint64_t *src = T(tags, q, rd.block);
          for (int w = 0; w < W; w++) {
            if (acc[w] & src[w]) throw InvalidArg("plan verification: duplicate contribution");
            acc[w] |= src[w];
          }
        }
        std::copy(acc.begin(), acc.end(), dst);
      }
    } else {
      for (const Transfer &t : st.transfers) {
        const uint64_t *src = T(tags, t.src, t.block);
        std::copy(src, src + W, T(nt, t.dst, t.block));
      }
    }
    tags.swap(nt);
  }
  for (int r = 0; r < n; r++)
    for (int b = 0; b < n; b++) {
      const uint64_t *v = T(tags, r, b);
      for (int w = 0; w < W; w++) {
        int bits = std::min(64, n - 64 * w);
        uint64_t full = bits == 64 ? ~0ull : ((1ull << bits) - 1);
        if (v[w] != full) throw InvalidArg("plan verification: missing contributions");
      }
    }
}

Plan plan_from_json(const std::string &text, std::string &dtype, bool &allreduce) {
  Json doc;
  try {
    doc = JsonReader(text).parse();
  } catch (const JsonError &e) {
    throw InvalidArg(e.what());
  }
  auto num = [](const Json *v, const char *what) -> long long {
    if (!v || v->kind != Json::Number || !v->is_integer) throw InvalidArg(std::string(what) + " must be an integer");
    return v->ival;
  };
  if (doc.kind != Json::Object) throw InvalidArg("plan must be an object");
  Plan p;
  p.n = (int)num(doc.get("n"), "n");
  p.count = num(doc.get("count"), "count");
  const Json *dt = doc.get("dtype");
  if (!dt || dt->kind != Json::String || (dt->str != "f32" && dt->str != "bf16")) throw InvalidArg("dtype must be f32|bf16");
  dtype = dt->str;
  if (p.n < 2 || p.n > 4096 || p.count < 1) throw InvalidArg("bad n/count");
  const Json *steps = doc.get("steps");
  if (!steps || steps->kind != Json::Array) throw InvalidArg("steps must be an array");
  if (const Json *sr = doc.get("switch_reduce")) {
    if (sr->kind != Json::Bool) throw InvalidArg("switch_reduce must be a boolean");
    p.switch_reduce = sr->b;
  }
  auto rank_ok = [&](long long r) {
    if (r < 0 || r >= p.n) throw InvalidArg("rank out of range");
    return (int)r;
  };
  for (const Json &sj : steps->arr) {
    if (sj.kind != Json::Object) throw InvalidArg("step must be an object");
    Step st;
    const Json *ph = sj.get("phase");
    if (!ph || ph->kind != Json::String || (ph->str != "rs" && ph->str != "ag")) throw InvalidArg("phase must be rs|ag");
    st.ag = ph->str == "ag";
    const Json *lb = sj.get("label");
    st.label = lb && lb->kind == Json::String ? lb->str : "";
    const Json *rds = sj.get("reduces");
    if (rds && rds->kind == Json::Array)
      for (const Json &rj : rds->arr) {
        Reduce rd;
        rd.server = rank_ok(num(rj.get("server"), "server"));
        rd.block = rank_ok(num(rj.get("block"), "block"));
        const Json *ins = rj.get("inputs");
        if (!ins || ins->kind != Json::Array || ins->arr.empty()) throw InvalidArg("reduce needs inputs");
        for (const Json &q : ins->arr) rd.inputs.push_back(rank_ok(num(&q, "input")));
        st.reduces.push_back(rd);
      }
    const Json *trs = sj.get("transfers");
    if (trs && trs->kind == Json::Array)
      for (const Json &tj : trs->arr) {
        Transfer t;
        t.src = rank_ok(num(tj.get("src"), "src"));
        t.dst = rank_ok(num(tj.get("dst"), "dst"));
        t.block = rank_ok(num(tj.get("block"), "block"));
        t.size = num(tj.get("size"), "size");
        if (t.size != block_size(p.count, p.n, t.block)) throw InvalidArg("transfer size != block size");
        if (t.src == t.dst) throw InvalidArg("transfer to itself");
        st.transfers.push_back(t);
      }
    if (st.ag && !st.reduces.empty()) throw InvalidArg("ag steps carry no reduces");
    if (!st.ag) add_implied_transfers(st, p.count, p.n);
    p.steps.push_back(std::move(st));
  }
  try {
    verify_allreduce(p);
    allreduce = true;
  } catch (const InvalidArg &e) {
    if (std::string(e.what()).find("hazard") != std::string::npos) throw;
    allreduce = false;
  }
  if (p.switch_reduce) check_switch_reduce(p);
  return p;
}

// A plan the executor's one-shot path can run with identical bits: two steps
// (RS, AG) whose RS step has one reduce per block, every reduce over all ranks in the same
// order.  Returns that order (empty: not eligible).
std::vector<int> oneshot_order(const Plan &P) {
  if (P.switch_reduce) return {};
  if (P.steps.size() != 2 || P.steps[0].ag || !P.steps[1].ag || (int)P.steps[0].reduces.size() != P.n) return {};
  const std::vector<int> &ord = P.steps[0].reduces[0].inputs;
  if ((int)ord.size() != P.n) return {};
  std::vector<char> seen(P.n, 0), blk(P.n, 0);
  for (int x : ord) {
    if (x < 0 || x >= P.n || seen[x]) return {};
    seen[x] = 1;
  }
  for (auto &rd : P.steps[0].reduces) {
    if (rd.inputs != ord || rd.block < 0 || rd.block >= P.n || blk[rd.block]) return {};
    blk[rd.block] = 1;
  }
  return ord;
}

// An NVLS plan is the single-switch CPS data movement: one RS step in which rank b
// reduces block b from all ranks, then its reversed AllGather.
void check_switch_reduce(const Plan &p) {
  const Plan want = build_plan_natural("cps", p.n, p.count);
  bool ok = p.steps.size() == want.steps.size();
  for (size_t i = 0; ok && i < p.steps.size(); i++) {
    const Step &a = p.steps[i], &b = want.steps[i];
    ok = a.ag == b.ag && a.reduces.size() == b.reduces.size() && a.transfers.size() == b.transfers.size();
    if (!ok) break;
    auto key_r = [](const Reduce &r) { return std::make_tuple(r.server, r.block, r.inputs); };
    auto key_t = [](const Transfer &t) { return std::make_tuple(t.dst, t.block, t.src); };
    std::vector<std::tuple<int, int, std::vector<int>>> ra, rb;
    for (auto &r : a.reduces) ra.push_back(key_r(r));
    for (auto &r : b.reduces) rb.push_back(key_r(r));
    std::vector<std::tuple<int, int, int>> ta, tb;
    for (auto &t : a.transfers) ta.push_back(key_t(t));
    for (auto &t : b.transfers) tb.push_back(key_t(t));
    std::sort(ra.begin(), ra.end());
    std::sort(rb.begin(), rb.end());
    std::sort(ta.begin(), ta.end());
    std::sort(tb.begin(), tb.end());
    ok = ra == rb && ta == tb;
  }
  if (!ok) throw InvalidArg("a switch_reduce (NVLS) plan must have the single-switch CPS data movement");
}

// ---------------------------------------------------------------- canonical JSON (O9)
std::string plan_to_json(const Plan &p, const char *dtype) {
  std::string o = "{\"count\":" + std::to_string(p.count) + ",\"dtype\":";
  json_escape(o, dtype);
  o += ",\"n\":" + std::to_string(p.n) + ",\"steps\":[";
  for (size_t si = 0; si < p.steps.size(); si++) {
    const Step &st = p.steps[si];
    if (si) o += ',';
    o += "{\"label\":";
    json_escape(o, st.label);
    o += ",\"phase\":";
    o += st.ag ? "\"ag\"" : "\"rs\"";
    o += ",\"reduces\":[";
    std::vector<const Reduce *> rds;
    for (auto &r : st.reduces) rds.push_back(&r);
    std::sort(rds.begin(), rds.end(), [](const Reduce *a, const Reduce *b) {
      return std::tie(a->server, a->block) < std::tie(b->server, b->block);
    });
    for (size_t i = 0; i < rds.size(); i++) {
      if (i) o += ',';
      o += "{\"block\":" + std::to_string(rds[i]->block) + ",\"fan_in\":" +
           std::to_string(rds[i]->inputs.size()) + ",\"inputs\":[";
      for (size_t k = 0; k < rds[i]->inputs.size(); k++) o += (k ? "," : "") + std::to_string(rds[i]->inputs[k]);
      o += "],\"server\":" + std::to_string(rds[i]->server) + "}";
    }
    o += "],\"transfers\":[";
    std::vector<const Transfer *> trs;
    for (auto &t : st.transfers) trs.push_back(&t);
    std::sort(trs.begin(), trs.end(), [](const Transfer *a, const Transfer *b) {
      return std::tie(a->dst, a->block, a->src) < std::tie(b->dst, b->block, b->src);
    });
    for (size_t i = 0; i < trs.size(); i++) {
      if (i) o += ',';
      o += "{\"block\":" + std::to_string(trs[i]->block) + ",\"dst\":" + std::to_string(trs[i]->dst) +
           ",\"size\":" + std::to_string(trs[i]->size) + ",\"src\":" + std::to_string(trs[i]->src) + "}";
    }
    o += "]}";
  }
  o += "]";
  if (p.switch_reduce) o += ",\"switch_reduce\":true";
  o += "}";
  return o;
}

static std::string fmt17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::string report_to_json(const std::vector<SwitchReport> &reps) {
  std::string o = "[";
  for (size_t i = 0; i < reps.size(); i++) {
    const SwitchReport &r = reps[i];
    if (i) o += ',';
    o += "{\"candidates\":[";
    for (size_t k = 0; k < r.candidates.size(); k++) {
      if (k) o += ',';
      o += "{\"kind\":";
      json_escape(o, r.candidates[k].first);
      o += ",\"total\":" + fmt17(r.candidates[k].second) + "}";
    }
    o += "],\"chosen\":";
    json_escape(o, r.chosen);
    o += ",\"finish_time\":" + fmt17(r.finish_time) + ",\"rearranged_children\":[";
    for (size_t k = 0; k < r.rearranged.size(); k++) {
      if (k) o += ',';
      json_escape(o, r.rearranged[k]);
    }
    o += "],\"start_time\":" + fmt17(r.start_time) + ",\"switch\":";
    json_escape(o, r.sw);
    o += "}";
  }
  return o + "]";
}

// ====================================================================== GenModel
std::vector<StepCoeffs> step_coeffs(const Plan &p, int esize) {
  std::vector<StepCoeffs> out;
  const int n = p.n;
  for (const Step &st : p.steps) {
    std::vector<int64_t> sent(n, 0), recv(n, 0), cc(n, 0), dd(n, 0);
    std::vector<std::set<int>> senders(n);
    for (const Transfer &t : st.transfers) {
      sent[t.src] += t.size * esize;
      recv[t.dst] += t.size * esize;
      senders[t.dst].insert(t.src);
    }
    for (const Reduce &rd : st.reduces) {
      int64_t k = (int64_t)rd.inputs.size();
      if (k >= 2) {
        int64_t sz = block_size(p.count, n, rd.block) * esize;
        cc[rd.server] += (k - 1) * sz;
        dd[rd.server] += (k + 1) * sz;
      }
    }
    StepCoeffs c;
    c.A = 1;
    c.B = std::max(*std::max_element(sent.begin(), sent.end()), *std::max_element(recv.begin(), recv.end()));
    c.C = *std::max_element(cc.begin(), cc.end());
    c.D = *std::max_element(dd.begin(), dd.end());
    size_t ms = 0;
    for (auto &s : senders) ms = std::max(ms, s.size());
    c.w = 1 + (int)ms;
    out.push_back(c);
  }
  return out;
}

std::vector<StepParams> uniform_step_params(const Params &p, size_t n) {
  double b, g;
  p.effective(b, g);
  return std::vector<StepParams>(n, StepParams{p.alpha, b, p.epsilon, p.w_t, g, p.delta});
}

static StepParams links_params(const Topology &t, const std::set<int> &links, double gamma, double delta) {
  if (links.empty()) return StepParams{0.0, 0.0, 0.0, 1 << 30, gamma, delta};
  double a = -1, b = -1, e = -1;
  int wt = std::numeric_limits<int>::max();
  for (int x : links) {
    const Uplink &u = t.nodes[x].up;
    a = std::max(a, u.alpha);
    b = std::max(b, u.beta);
    e = std::max(e, u.epsilon);
    wt = std::min(wt, u.w_t);
  }
  return StepParams{a, b / 4, e / 4, wt, gamma, delta};
}

std::vector<StepParams> topo_step_params(const Topology &t, const Plan &p) {
  double g = -1, d = -1;
  for (int s : t.servers) {
    g = std::max(g, t.nodes[s].comp.gamma);
    d = std::max(d, t.nodes[s].comp.delta);
  }
  g = g / 4;
  d = d / 4;
  std::vector<StepParams> out;
  for (const Step &st : p.steps) {
    std::set<int> links;
    for (const Transfer &tr : st.transfers)
      for (int x : t.path_links(t.servers[tr.src], t.servers[tr.dst])) links.insert(x);
    out.push_back(links_params(t, links, g, d));
  }
  return out;
}

Breakdown predict_f64(const std::vector<StepCoeffs> &cs, const std::vector<StepParams> &ps) {
  Breakdown r;
  for (size_t i = 0; i < cs.size(); i++) {
    const StepCoeffs &c = cs[i];
    const StepParams &p = ps[i];
    double a = (double)c.A * p.alpha;
    double b = (double)c.B * p.beta;
    double g = (double)c.C * p.gamma;
    double d = (double)c.D * p.delta;
    int64_t ex = c.w - p.w_t > 0 ? (int64_t)(c.w - p.w_t) : 0;
    double in = (double)(ex * c.B) * p.epsilon;
    double t = (((a + b) + g) + d) + in;
    r.latency += a;
    r.bandwidth += b;
    r.compute += g;
    r.memory += d;
    r.incast += in;
    r.total += t;
  }
  return r;
}

// Table 2 rows with readings Q5/Q6/Q7 as integer numerators over `den`.
static void closed_form_terms(const std::string &kind, int c, int64_t S, int w_t, const std::vector<int> &f,
                              int64_t &A, int64_t &Bn, int64_t &Cn, int64_t &Dn, int64_t &In, int64_t &den) {
  if (c < 2) throw InvalidArg("closed forms need N >= 2");
  const int64_t cm1 = c - 1;
  const int64_t over = c - w_t > 0 ? c - w_t : 0;
  if (kind == "rb") {
    A = 2; Bn = 2 * cm1 * S; Cn = cm1 * S; Dn = (int64_t)(c + 1) * S; In = 2 * cm1 * S * over; den = 1;
  } else if (kind == "cps") {
    A = 2; Bn = 2 * cm1 * S; Cn = cm1 * S; Dn = (int64_t)(c + 1) * S; In = 2 * cm1 * S * over; den = c;
  } else if (kind == "ring") {
    A = 2 * cm1; Bn = 2 * cm1 * S; Cn = cm1 * S; Dn = 3 * cm1 * S; In = 0; den = c;
  } else if (kind == "rhd") {
    int64_t chi = is_pow2(c) ? 0 : 1;
    A = 2 * ceil_log2(c); Bn = 2 * cm1 * S + chi * 2 * S * c; Cn = cm1 * S + chi * S * c;
    Dn = 3 * cm1 * S + chi * 3 * S * c; In = 0; den = c;
  } else if (kind == "hcps") {
    int64_t prod = 1;
    for (int x : f) prod *= x;
    bool bad = f.empty() || prod != c;
    for (int x : f) bad = bad || x < 2;
    if (bad) throw InvalidArg("invalid hcps factorization");
    const int m = (int)f.size();
    int64_t suffix = 0;
    for (int i = 1; i < m; i++) {
      int64_t p = 1;
      for (int j = i; j < m; j++) p *= f[j];
      suffix += p;
    }
    int64_t inc = 0;
    for (int i = 0; i < m; i++) {
      int64_t tail = 1;
      for (int j = i + 1; j < m; j++) tail *= f[j];
      int64_t ov = f[i] - w_t > 0 ? f[i] - w_t : 0;
      inc += ov * 2 * (f[i] - 1) * tail;
    }
    A = 2 * m; Bn = 2 * cm1 * S; Cn = cm1 * S; Dn = (2 * suffix + c + 1) * S; In = inc * S; den = c;
  } else if (kind == "nvls") {
    // DESIGN.md reading NV1: in-switch fan-in-N reduce + multicast; (N+1)S/N per direction
    A = 2; Bn = (int64_t)(c + 1) * S; Cn = 0; Dn = 0; In = 0; den = c;
  } else if (kind == "oneshot") {
    // DESIGN.md reading OS1: the executor's one-shot small-message path
    A = 1; Bn = 2 * cm1 * S; Cn = cm1 * S; Dn = (int64_t)(c + 1) * S; In = 2 * cm1 * S * over; den = 1;
  } else if (kind == "ll128") {
    // the executor's LL128 two-shot path: 128-byte lines of 120 payload bytes, one round
    A = 1; Bn = 32 * cm1 * S; Cn = 15 * cm1 * S; Dn = 15 * (int64_t)(c + 1) * S; In = 32 * cm1 * S * over;
    den = 15 * (int64_t)c;
  } else {
    throw InvalidArg("no closed form for " + kind);
  }
}

Breakdown closed_form_f64(const std::string &kind, int c, int64_t S, const Params &p, const std::vector<int> &f) {
  int64_t A, Bn, Cn, Dn, In, den;
  closed_form_terms(kind, c, S, p.w_t, f, A, Bn, Cn, Dn, In, den);
  double beta, gamma;
  p.effective(beta, gamma);
  const double dd = (double)den;
  Breakdown r;
  r.latency = (double)A * p.alpha;
  r.bandwidth = ((double)Bn / dd) * beta;
  r.compute = ((double)Cn / dd) * gamma;
  r.memory = ((double)Dn / dd) * p.delta;
  r.incast = ((double)In / dd) * p.epsilon;
  r.total = (((r.latency + r.bandwidth) + r.compute) + r.memory) + r.incast;
  return r;
}

std::vector<std::vector<int>> hcps_factorizations(int n, int max_steps) {
  std::vector<std::vector<int>> found;
  std::vector<int> pref;
  std::function<void(int)> rec = [&](int rem) {
    if (rem == 1) {
      if (!pref.empty()) found.push_back(pref);
      return;
    }
    if ((int)pref.size() == max_steps) return;
    for (int d = 2; d <= rem; d++)
      if (rem % d == 0) {
        pref.push_back(d);
        rec(rem / d);
        pref.pop_back();
      }
  };
  rec(n);
  std::vector<std::vector<int>> out;
  for (int m = 1; m <= max_steps; m++) {
    std::vector<std::vector<int>> lm;
    for (auto &f : found)
      if ((int)f.size() == m) lm.push_back(f);
    std::sort(lm.begin(), lm.end(), std::greater<std::vector<int>>());
    out.insert(out.end(), lm.begin(), lm.end());
  }
  return out;
}

// ====================================================================== GenTree
namespace {

struct Cand { std::string name; std::vector<int> f; };

static std::vector<Cand> candidates_for(int c) {   // reading Q13, tie-break order
  std::vector<Cand> out{{"cps", {}}};
  for (auto &f : hcps_factorizations(c, 3))
    if (f.size() >= 2) out.push_back({"hcps", f});
  if (is_pow2(c)) out.push_back({"rhd", {}});
  out.push_back({"ring", {}});
  return out;
}

static int steps_of(const std::string &name, int c, const std::vector<int> &f) {
  if (name == "cps" || name == "rb") return 2;
  if (name == "ring") return 2 * (c - 1);
  if (name == "rhd") return 2 * ceil_log2(c);
  return 2 * (int)f.size();
}

static int f0_of(const std::string &name, int c, const std::vector<int> &f) {
  if (name == "cps") return c;
  if (name == "hcps") return f[0];
  return 2;
}

static double step_cost(const StepCoeffs &c, const StepParams &p) {
  return predict_f64({c}, {p}).total;
}

// ACPS (P:629 footnote): every block not at its final owner goes straight there.
static std::vector<Step> build_acps(const std::map<int, std::set<int>> &init,
                                    const std::vector<std::pair<int, std::vector<int>>> &final_place,
                                    int64_t count, int n, const std::string &label) {
  std::map<int, std::vector<int>> holders;
  for (auto &kv : init)
    for (int b : kv.second) holders[b].push_back(kv.first);
  std::map<int, int> owner;
  for (auto &kv : final_place)
    for (int b : kv.second) {
      if (owner.count(b)) throw InvalidArg("block has two owners");
      owner[b] = kv.first;
    }
  if (owner.size() != holders.size()) throw InvalidArg("placements cover different blocks");
  for (auto &kv : owner)
    if (!holders.count(kv.first)) throw InvalidArg("placements cover different blocks");
  Step st;
  st.label = label;
  for (auto &kv : owner) {
    std::vector<int> hs = holders[kv.first];
    std::sort(hs.begin(), hs.end());
    if (hs.size() == 1 && hs[0] == kv.second) continue;
    st.reduces.push_back({kv.second, kv.first, hs});
  }
  if (st.reduces.empty()) return {};
  add_implied_transfers(st, count, n);
  return {st};
}

}  // namespace

PlanResult gentree(const Topology &t, int64_t count, int esize, const Params *explicit_params,
                   const std::string &force_in) {
  // "norearrange": GenTree* of tab:gentreesimu ("the special plan without data
  // rearrangement") — Algorithm 2 with the data-rearrangement optimisation switched off
  const bool rearrange = force_in != "norearrange";
  const std::string force = rearrange ? force_in : std::string();
  const int N = (int)t.servers.size();
  if (count < 1) throw InvalidArg("count must be >= 1");
  const int64_t S = count * esize;
  PlanResult res;
  std::string fname;
  std::vector<int> ff;
  if (!force.empty()) {
    parse_kind(force, fname, ff);
    if (fname == "rb") {
      for (int c : t.nodes[t.root].children)
        if (!t.nodes[c].server) throw InvalidArg("rb is only defined on a single-switch topology");
      res.plan = build_plan_natural("rb", N, count);
      verify_allreduce(res.plan);
      SwitchReport r;
      r.sw = t.nodes[t.root].id;
      r.chosen = "rb";
      res.reports.push_back(r);
      return res;
    }
  }
  const size_t NN = t.nodes.size();
  // ---- Algorithm 1: final placement per node (ordered rank -> blocks)
  std::vector<std::vector<std::pair<int, std::vector<int>>>> basic(NN);
  std::function<void(int)> alg1 = [&](int nid) {
    const Node &nd = t.nodes[nid];
    if (nd.server) {
      std::vector<int> all(N);
      std::iota(all.begin(), all.end(), 0);
      basic[nid] = {{nd.rank, all}};
      return;
    }
    for (int ch : nd.children) alg1(ch);
    std::vector<char> taken(N, 0);
    std::vector<int> under;
    t.servers_under(nid, under);
    const int n = (int)under.size();
    const int num_blocks = N / n;
    int remain = N % n;
    std::vector<std::pair<int, std::vector<int>>> place;
    std::vector<int> quota;
    for (int ch : nd.children)
      for (auto &sb : basic[ch]) {
        int want = num_blocks;
        if (remain > 0) { want += 1; remain -= 1; }
        std::vector<int> got;
        for (int b : sb.second)
          if (!taken[b]) {
            taken[b] = 1;
            got.push_back(b);
            if (--want == 0) break;
          }
        place.push_back({sb.first, got});
        quota.push_back(want);
      }
    for (int b = 0; b < N; b++)        // reading Q12: complete the partition
      if (!taken[b])
        for (size_t i = 0; i < place.size(); i++)
          if (quota[i] > 0) {
            place[i].second.push_back(b);
            quota[i]--;
            taken[b] = 1;
            break;
          }
    basic[nid] = place;
  };
  alg1(t.root);

  // ---- Algorithm 2
  std::vector<std::vector<Step>> local(NN);
  std::vector<double> finish(NN, 0.0);
  std::vector<std::map<int, std::set<int>>> place_now(NN);
  auto uplink_sp = [&](int nid) -> StepParams {
    if (explicit_params) return uniform_step_params(*explicit_params, 1)[0];
    const Uplink &u = t.nodes[nid].up;
    return StepParams{u.alpha, u.beta / 4, u.epsilon / 4, u.w_t, 0.0, 0.0};
  };
  auto switch_params = [&](int nid) -> Params {
    if (explicit_params) return *explicit_params;
    std::vector<int> sub;
    t.subtree(nid, sub);
    Params p;
    double a = -1, b = -1, e = -1, g = -1, d = -1;
    int wt = std::numeric_limits<int>::max();
    for (int x : sub) {
      if (x == nid) continue;
      const Uplink &u = t.nodes[x].up;
      a = std::max(a, u.alpha);
      b = std::max(b, u.beta);
      e = std::max(e, u.epsilon);
      wt = std::min(wt, u.w_t);
      if (t.nodes[x].server) {
        g = std::max(g, t.nodes[x].comp.gamma);
        d = std::max(d, t.nodes[x].comp.delta);
      }
    }
    p.alpha = a; p.beta = b / 4; p.gamma = g / 4; p.delta = d / 4; p.epsilon = e / 4; p.w_t = wt;
    return p;
  };

  std::function<void(int)> alg2 = [&](int nid) {
    const Node &nd = t.nodes[nid];
    if (nd.server) {
      std::set<int> all;
      for (int b = 0; b < N; b++) all.insert(b);
      place_now[nid][nd.rank] = all;
      return;
    }
    for (int ch : nd.children) alg2(ch);
    std::vector<int> own(N, -1);
    for (auto &sb : basic[nid])
      for (int b : sb.second) own[b] = sb.first;
    SwitchReport rep;
    rep.sw = nd.id;
    // ---- data rearrangement (readings Q15/Q15b)
    for (int ch : nd.children) {
      if (!rearrange || t.nodes[ch].server) continue;
      std::vector<int> chs;
      t.servers_under(ch, chs);
      const int ni = (int)chs.size();
      if (ni < 2) continue;
      int k = t.rearrangement_subset_size(nid, ch, ni);   // ceil(n_i / r), exact (Q15)
      k = std::max(1, std::min(ni, k));
      if (k >= ni) continue;
      std::vector<int> subset(chs.begin(), chs.begin() + k);
      const auto &cur = place_now[ch];
      std::vector<std::pair<int, int>> held;   // (block, rank)
      for (auto &kv : cur)
        for (int b : kv.second) held.push_back({b, kv.first});
      std::sort(held.begin(), held.end());
      std::map<int, std::set<int>> rearr;
      for (int r : chs) rearr[r];
      std::vector<std::tuple<int, int, int>> moves;   // (src, dst, block)
      for (size_t j = 0; j < held.size(); j++) {
        int dst = subset[j % k];
        rearr[dst].insert(held[j].first);
        if (dst != held[j].second) moves.emplace_back(held[j].second, dst, held[j].first);
      }
      std::set<int> chset(chs.begin(), chs.end());
      auto out_time = [&](const std::map<int, std::set<int>> &pl) {
        int64_t B = 0;
        std::set<int> senders;
        for (auto &kv : pl)
          for (int b : kv.second)
            if (!chset.count(own[b])) {
              B += block_size(count, N, b) * esize;
              senders.insert(kv.first);
            }
        return step_cost(StepCoeffs{1, B, 0, 0, (int)senders.size()}, uplink_sp(ch));
      };
      double t_origin = out_time(cur);
      std::map<int, int64_t> sent, recv;
      std::map<int, std::set<int>> snd;
      for (auto &mv : moves) {
        int64_t sz = block_size(count, N, std::get<2>(mv)) * esize;
        sent[std::get<0>(mv)] += sz;
        recv[std::get<1>(mv)] += sz;
        snd[std::get<1>(mv)].insert(std::get<0>(mv));
      }
      int64_t Bm = 0;
      for (auto &kv : sent) Bm = std::max(Bm, kv.second);
      for (auto &kv : recv) Bm = std::max(Bm, kv.second);
      size_t ws = 0;
      for (auto &kv : snd) ws = std::max(ws, kv.second.size());
      StepParams sp;
      if (explicit_params) {
        sp = uniform_step_params(*explicit_params, 1)[0];
      } else {
        std::set<int> links;
        for (auto &mv : moves)
          for (int x : t.path_links(t.servers[std::get<0>(mv)], t.servers[std::get<1>(mv)])) links.insert(x);
        sp = links_params(t, links, 0.0, 0.0);
      }
      double t_cps = step_cost(StepCoeffs{1, Bm, 0, 0, 1 + (int)ws}, sp);
      double t_rearr = t_cps + out_time(rearr);
      if (!moves.empty() && t_rearr < t_origin) {
        Step st;
        st.label = t.nodes[ch].id + ":rearrange";
        std::stable_sort(moves.begin(), moves.end(),
                         [](const std::tuple<int, int, int> &a, const std::tuple<int, int, int> &b) {
                           return std::get<2>(a) < std::get<2>(b);
                         });
        for (auto &mv : moves) st.reduces.push_back({std::get<1>(mv), std::get<2>(mv), {std::get<0>(mv)}});
        local[ch].push_back(st);
        finish[ch] += t_cps;
        place_now[ch] = rearr;
        rep.rearranged.push_back(t.nodes[ch].id);
      }
    }
    double start = -std::numeric_limits<double>::infinity();
    for (int ch : nd.children) start = std::max(start, finish[ch]);
    // ---- plan-type selection
    std::map<int, std::set<int>> init;
    for (int ch : nd.children)
      for (auto &kv : place_now[ch]) init[kv.first].insert(kv.second.begin(), kv.second.end());
    std::vector<std::vector<int>> holders(N);
    for (auto &kv : init)                 // std::map iterates ranks ascending
      for (int b : kv.second) holders[b].push_back(kv.first);
    const int c = (int)nd.children.size();
    std::set<int> counts;
    for (int ch : nd.children) {
      std::vector<int> u;
      t.servers_under(ch, u);
      counts.insert((int)u.size());
    }
    bool regular = counts.size() == 1;
    for (int b = 0; regular && b < N; b++)
      regular = (int)holders[b].size() == c &&
                std::find(holders[b].begin(), holders[b].end(), own[b]) != holders[b].end();
    Params spx = switch_params(nid);
    std::vector<Cand> cands;
    if (c == 1) {
      rep.chosen = "none";
    } else if (regular) {
      cands = candidates_for(c);
      if (!force.empty()) {
        if (fname == "hcps") {
          int64_t p = 1;
          bool bad = false;
          for (int x : ff) { p *= x; bad = bad || x < 2; }
          if (bad || p != c) throw InvalidArg("hcps fan-ins do not multiply to the child count at switch " + nd.id);
        }
        if (fname == "rhd" && !is_pow2(c)) throw InvalidArg("rhd needs a power-of-two child count at " + nd.id);
        cands = {{fname, ff}};
      }
    } else {
      cands = {{"acps", {}}};
    }
    std::vector<std::pair<int, std::vector<int>>> final_place = basic[nid];
    bool have_best = false;
    std::tuple<double, int, int, int> best_key;
    Cand best;
    double best_total = 0;
    for (size_t idx = 0; idx < cands.size(); idx++) {
      const Cand &cd = cands[idx];
      double total;
      int nst;
      if (cd.name == "acps") {
        auto st = build_acps(init, final_place, count, N, nd.id + ":acps");
        Plan tmp;
        tmp.n = N;
        tmp.count = count;
        tmp.steps = st;
        auto ag = reverse_to_allgather(st);
        tmp.steps.insert(tmp.steps.end(), ag.begin(), ag.end());
        auto co = step_coeffs(tmp, esize);
        total = predict_f64(co, uniform_step_params(spx, co.size())).total;
        nst = (int)co.size();
      } else {
        total = closed_form_f64(cd.name, c, S, spx, cd.f).total;
        nst = steps_of(cd.name, c, cd.f);
      }
      rep.candidates.push_back({kind_label(cd.name, cd.f), total});
      auto key = std::make_tuple(total, nst, -f0_of(cd.name, c, cd.f), (int)idx);
      if (!have_best || key < best_key) {
        have_best = true;
        best_key = key;
        best = cd;
        best_total = total;
      }
    }
    std::vector<Step> steps;
    if (have_best) {
      rep.chosen = kind_label(best.name, best.f);
      if (best.name == "acps") {
        steps = build_acps(init, final_place, count, N, nd.id + ":acps");
      } else {
        std::map<std::vector<int>, std::vector<int>> groups;
        for (int b = 0; b < N; b++) groups[holders[b]].push_back(b);
        std::vector<std::pair<std::vector<int>, std::vector<int>>> glist(groups.begin(), groups.end());
        std::sort(glist.begin(), glist.end(),
                  [](const std::pair<std::vector<int>, std::vector<int>> &a,
                     const std::pair<std::vector<int>, std::vector<int>> &b) { return a.second[0] < b.second[0]; });
        std::vector<int> natowner;
        auto nat = natural_rs(best.name, c, best.f, natowner);
        std::string lab = nd.id + ":" + kind_label(best.name, best.f);
        for (auto &g : glist) {
          const std::vector<int> &tup = g.first;
          std::vector<std::vector<int>> chunk_of(c);
          for (int k = 0; k < c; k++)
            for (int b : g.second)
              if (own[b] == tup[k]) chunk_of[k].push_back(b);
          std::vector<std::vector<int>> chunk_blocks(c);
          for (int j = 0; j < c; j++) chunk_blocks[j] = chunk_of[natowner[j]];
          auto gst = realize(nat, chunk_blocks, tup, lab);
          for (size_t i = 0; i < gst.size(); i++) {
            if (i == steps.size()) {
              Step s;
              s.label = lab;
              steps.push_back(s);
            }
            steps[i].reduces.insert(steps[i].reduces.end(), gst[i].reduces.begin(), gst[i].reduces.end());
          }
        }
      }
      rep.finish_time = start + best_total;
    } else {
      rep.finish_time = start;
    }
    rep.start_time = start;
    local[nid] = steps;
    finish[nid] = rep.finish_time;
    place_now[nid].clear();
    for (auto &sb : basic[nid]) place_now[nid][sb.first] = std::set<int>(sb.second.begin(), sb.second.end());
    res.reports.push_back(rep);
  };
  alg2(t.root);

  // ---- composition: global index = max over children of (start + length)
  std::vector<int> start_idx(NN, 0), length(NN, 0);
  std::function<void(int)> sched = [&](int nid) {
    const Node &nd = t.nodes[nid];
    if (nd.server) return;
    int s = 0;
    for (int ch : nd.children) {
      sched(ch);
      s = std::max(s, start_idx[ch] + length[ch]);
    }
    start_idx[nid] = s;
    length[nid] = (int)local[nid].size();
  };
  sched(t.root);
  const int total_rs = start_idx[t.root] + length[t.root];
  std::vector<Step> rs(total_rs);
  std::vector<std::vector<std::string>> labels(total_rs);
  std::function<void(int)> compose = [&](int nid) {
    const Node &nd = t.nodes[nid];
    if (nd.server) return;
    for (int ch : nd.children) compose(ch);
    for (size_t i = 0; i < local[nid].size(); i++) {
      int g = start_idx[nid] + (int)i;
      rs[g].reduces.insert(rs[g].reduces.end(), local[nid][i].reduces.begin(), local[nid][i].reduces.end());
      labels[g].push_back(local[nid][i].label);
    }
  };
  compose(t.root);
  std::vector<Step> steps;
  for (int g = 0; g < total_rs; g++) {
    if (rs[g].reduces.empty()) continue;
    std::string lab;
    for (size_t i = 0; i < labels[g].size(); i++) lab += (i ? "+" : "") + labels[g][i];
    rs[g].label = lab;
    add_implied_transfers(rs[g], count, N);
    steps.push_back(rs[g]);
  }
  res.plan.n = N;
  res.plan.count = count;
  res.plan.steps = steps;
  auto ag = reverse_to_allgather(steps);
  res.plan.steps.insert(res.plan.steps.end(), ag.begin(), ag.end());
  verify_allreduce(res.plan);
  return res;
}

// ====================================================================== fit
// Lawson-Hanson NNLS for small dense problems (m rows, n <= 8 columns).
static std::vector<double> nnls(const std::vector<std::vector<double>> &A, const std::vector<double> &b) {
  const size_t m = A.size(), n = A[0].size();
  std::vector<double> x(n, 0.0);
  std::vector<char> P(n, 0);
  auto lsq_on = [&](const std::vector<char> &set, std::vector<double> &z) {
    // normal equations on the passive set (n <= 8; columns are pre-scaled)
    std::vector<int> idx;
    for (size_t j = 0; j < n; j++)
      if (set[j]) idx.push_back((int)j);
    const size_t k = idx.size();
    std::vector<double> M(k * k, 0.0), v(k, 0.0);
    for (size_t i = 0; i < m; i++)
      for (size_t a = 0; a < k; a++) {
        v[a] += A[i][idx[a]] * b[i];
        for (size_t c = 0; c < k; c++) M[a * k + c] += A[i][idx[a]] * A[i][idx[c]];
      }
    // Gaussian elimination with partial pivoting
    for (size_t col = 0; col < k; col++) {
      size_t piv = col;
      for (size_t r = col + 1; r < k; r++)
        if (std::fabs(M[r * k + col]) > std::fabs(M[piv * k + col])) piv = r;
      for (size_t c = 0; c < k; c++) std::swap(M[col * k + c], M[piv * k + c]);
      std::swap(v[col], v[piv]);
      double d = M[col * k + col];
      if (d == 0.0) continue;
      for (size_t r = col + 1; r < k; r++) {
        double fct = M[r * k + col] / d;
        for (size_t c = col; c < k; c++) M[r * k + c] -= fct * M[col * k + c];
        v[r] -= fct * v[col];
      }
    }
    std::vector<double> sol(k, 0.0);
    for (size_t r = k; r-- > 0;) {
      double s = v[r];
      for (size_t c = r + 1; c < k; c++) s -= M[r * k + c] * sol[c];
      sol[r] = M[r * k + r] != 0.0 ? s / M[r * k + r] : 0.0;
    }
    z.assign(n, 0.0);
    for (size_t a = 0; a < k; a++) z[idx[a]] = sol[a];
  };
  for (int outer = 0; outer < 3 * (int)n + 10; outer++) {
    std::vector<double> w(n, 0.0);
    for (size_t j = 0; j < n; j++) {
      double s = 0;
      for (size_t i = 0; i < m; i++) {
        double r = b[i];
        for (size_t c = 0; c < n; c++) r -= A[i][c] * x[c];
        s += A[i][j] * r;
      }
      w[j] = s;
    }
    int jmax = -1;
    double wmax = 1e-14;
    for (size_t j = 0; j < n; j++)
      if (!P[j] && w[j] > wmax) { wmax = w[j]; jmax = (int)j; }
    if (jmax < 0) break;
    P[jmax] = 1;
    for (int inner = 0; inner < 3 * (int)n + 10; inner++) {
      std::vector<double> z;
      lsq_on(P, z);
      bool ok = true;
      for (size_t j = 0; j < n; j++)
        if (P[j] && z[j] <= 0) ok = false;
      if (ok) { x = z; break; }
      double alpha = 1.0;
      for (size_t j = 0; j < n; j++)
        if (P[j] && z[j] <= 0) alpha = std::min(alpha, x[j] / (x[j] - z[j]));
      for (size_t j = 0; j < n; j++) x[j] += alpha * (z[j] - x[j]);
      for (size_t j = 0; j < n; j++)
        if (P[j] && x[j] <= 1e-300) { P[j] = 0; x[j] = 0; }
    }
  }
  return x;
}

FitResult fit_params(const std::vector<Measurement> &rows_in, int wt_min, int wt_max) {
  std::map<std::pair<int, double>, std::vector<double>> acc;
  for (auto &r : rows_in) acc[{r.n, r.s}].push_back(r.t);
  std::vector<Measurement> rows;
  std::set<int> ns;
  std::set<double> ss;
  for (auto &kv : acc) {
    double sum = 0;
    for (double v : kv.second) sum += v;
    rows.push_back({kv.first.first, kv.first.second, sum / kv.second.size()});
    ns.insert(kv.first.first);
    ss.insert(kv.first.second);
  }
  if (rows.size() < 4) throw InvalidArg("underdetermined: need >= 4 distinct (n, s) rows");
  if (ns.size() < 2 || ss.size() < 2) throw InvalidArg("underdetermined: need >= 2 distinct n and >= 2 distinct s");
  if (wt_min < 1 || wt_max < wt_min) throw InvalidArg("bad w_t range");
  struct Cand { int wt; double sse; std::vector<double> x; };
  std::vector<Cand> scan;
  for (int wt = wt_min; wt <= wt_max; wt++) {
    std::vector<std::vector<double>> A;
    std::vector<double> b;
    for (auto &r : rows) {
      double n = r.n, s = r.s;
      A.push_back({2.0, (n - 1) * s / n, (n + 1) * s / n, std::max(r.n - wt, 0) * 2.0 * (n - 1) * s / n});
      b.push_back(r.t);
    }
    std::vector<double> scale(4, 0.0);
    for (auto &row : A)
      for (int j = 0; j < 4; j++) scale[j] = std::max(scale[j], std::fabs(row[j]));
    for (int j = 0; j < 4; j++) scale[j] = std::max(scale[j], 1e-300);
    auto As = A;
    for (auto &row : As)
      for (int j = 0; j < 4; j++) row[j] /= scale[j];
    auto x = nnls(As, b);
    for (int j = 0; j < 4; j++) x[j] /= scale[j];
    double sse = 0;
    for (size_t i = 0; i < A.size(); i++) {
      double r = -b[i];
      for (int j = 0; j < 4; j++) r += A[i][j] * x[j];
      sse += r * r;
    }
    scan.push_back({wt, sse, x});
  }
  double best = scan[0].sse;
  for (auto &c : scan) best = std::min(best, c.sse);
  double tol = best * 1e-6 + 1e-24;
  for (auto &c : scan)
    if (c.sse <= best + tol) {
      FitResult f;
      f.alpha = c.x[0];
      f.combined = c.x[1];
      f.delta = c.x[2];
      f.epsilon = c.x[3];
      f.w_t = c.wt;
      f.sse = c.sse;
      return f;
    }
  throw InvalidArg("fit failed");
}

NvlsFit fit_nvls(const std::vector<Measurement> &rows_in) { return fit_row("nvls", rows_in); }

NvlsFit fit_row(const std::string &kind, const std::vector<Measurement> &rows_in) {
  std::map<std::pair<int, double>, std::vector<double>> acc;
  for (auto &r : rows_in) acc[{r.n, r.s}].push_back(r.t);
  std::vector<Measurement> rows;
  std::set<double> ss;
  for (auto &kv : acc) {
    double sum = 0;
    for (double v : kv.second) sum += v;
    rows.push_back({kv.first.first, kv.first.second, sum / kv.second.size()});
    ss.insert(kv.first.second);
  }
  if (rows.size() < 2 || ss.size() < 2) throw InvalidArg("underdetermined: need >= 2 distinct sizes");
  std::vector<std::vector<double>> A;
  std::vector<double> b;
  for (auto &r : rows) {
    int64_t a_, bn, cn, dn, in, den;
    closed_form_terms(kind, r.n, (int64_t)r.s, 1 << 30, {}, a_, bn, cn, dn, in, den);
    A.push_back({(double)a_, (double)bn / (double)den});
    b.push_back(r.t);
  }
  double scale[2] = {1e-300, 1e-300};
  for (auto &row : A)
    for (int j = 0; j < 2; j++) scale[j] = std::max(scale[j], std::fabs(row[j]));
  auto As = A;
  for (auto &row : As)
    for (int j = 0; j < 2; j++) row[j] /= scale[j];
  auto x = nnls(As, b);
  for (int j = 0; j < 2; j++) x[j] /= scale[j];
  NvlsFit f;
  f.alpha = x[0];
  f.beta = x[1];
  for (size_t i = 0; i < A.size(); i++) {
    double r = A[i][0] * x[0] + A[i][1] * x[1] - b[i];
    f.sse += r * r;
  }
  return f;
}

}  // namespace gtar
