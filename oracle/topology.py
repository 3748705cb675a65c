"""Tree topology (oracle; test infrastructure only).

PAPER.md P:562-563 ("each tree-based physical topology has a root node, and every non-root
node has a link connecting to its parent ... The leaves of a tree are servers ... Other
non-leaf nodes are switches"), Table 5 for the per-level parameters.
The document format is SPEC.md's: {"nodes": [{id, kind, parent, uplink, compute}]}.

Link parameters live on the child side of each edge ("uplink"); β, γ, δ, ε in the
document are per 4-byte float (Table 5 units).  Ranks are the servers in depth-first
pre-order with children in document order (reading R1).
"""
from __future__ import annotations

from fractions import Fraction

import json
from dataclasses import dataclass, field

UPLINK_KEYS = {"alpha", "beta", "epsilon", "w_t"}
COMPUTE_KEYS = {"gamma", "delta"}
NODE_KEYS = {"id", "kind", "parent", "uplink", "compute"}


class TopologyError(ValueError):
    """Validation error (SPEC exit code 1)."""


@dataclass
class Node:
    id: str
    kind: str                       # "switch" | "server"
    parent: str | None
    uplink: dict | None             # alpha s, beta s/float, epsilon s/float, w_t int
    compute: dict | None            # gamma s/float, delta s/float
    children: list = field(default_factory=list)


@dataclass
class Topology:
    nodes: dict                     # id -> Node, document order
    root: str
    servers: list                   # DFS pre-order; rank r = servers[r]
    rank: dict                      # server id -> rank

    def servers_under(self, nid: str) -> list:
        """All server leaves under `nid` in DFS order (Alg. 1 num_servers)."""
        if nid not in self.nodes:
            raise TopologyError(f"unknown node {nid!r}")
        out = []

        def dfs(x):
            n = self.nodes[x]
            if n.kind == "server":
                out.append(x)
            for c in n.children:
                dfs(c)
        dfs(nid)
        return out

    def ranks_under(self, nid: str) -> list:
        return [self.rank[s] for s in self.servers_under(nid)]

    def subtree(self, nid: str) -> list:
        out = []

        def dfs(x):
            out.append(x)
            for c in self.nodes[x].children:
                dfs(c)
        dfs(nid)
        return out

    def path_links(self, a: str, b: str) -> list:
        """Nodes whose uplink a transfer a->b traverses: up to the LCA, then down."""
        up_a = [a]
        while self.nodes[up_a[-1]].parent is not None:
            up_a.append(self.nodes[up_a[-1]].parent)
        up_b = [b]
        while self.nodes[up_b[-1]].parent is not None:
            up_b.append(self.nodes[up_b[-1]].parent)
        sa = set(up_a)
        lca = next(x for x in up_b if x in sa)
        return up_a[:up_a.index(lca)] + up_b[:up_b.index(lca)]

    def convergence_ratio(self, switch: str, child: str) -> Fraction:
        """P:626 "the total bandwidth of A to its children divided by that of C_i",
        exactly: r = β_i · Σ_k 1/β_k over A's children, as a rational of the given floats."""
        sw = self.nodes[switch]
        if child not in sw.children:
            raise TopologyError(f"{child!r} is not a child of {switch!r}")
        inv = sum(Fraction(1) / Fraction(self.nodes[c].uplink["beta"]) for c in sw.children)
        return Fraction(self.nodes[child].uplink["beta"]) * inv

    def convergence_ratio_f64(self, switch: str, child: str) -> float:
        """P:626 "the total bandwidth of A to its children divided by that of C_i".

        Evaluated in float64 in a fixed order (reading Q15b) so the library and
        the oracle round identically: beta_i * sum_k (1/beta_k), children in document order.
        """
        sw = self.nodes[switch]
        if child not in sw.children:
            raise TopologyError(f"{child!r} is not a child of {switch!r}")
        acc = 0.0
        for c in sw.children:
            acc = acc + 1.0 / self.nodes[c].uplink["beta"]
        return self.nodes[child].uplink["beta"] * acc


def _num(v, what):
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise TopologyError(f"{what} must be a number")
    return float(v)


def parse_topology(text: str) -> Topology:
    """parse + validate a topology document; raises TopologyError."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise TopologyError(f"syntax error: {e}") from None
    if not isinstance(doc, dict) or set(doc) != {"nodes"} or not isinstance(doc["nodes"], list):
        raise TopologyError('top level must be {"nodes": [...]}')
    nodes = {}
    for nd in doc["nodes"]:
        if not isinstance(nd, dict):
            raise TopologyError("node must be an object")
        extra = set(nd) - NODE_KEYS
        if extra:
            raise TopologyError(f"unknown keys {sorted(extra)}")
        nid = nd.get("id")
        if not isinstance(nid, str) or not nid:
            raise TopologyError("node id must be a non-empty string")
        if nid in nodes:
            raise TopologyError(f"duplicate id {nid!r}")
        kind = nd.get("kind")
        if kind not in ("switch", "server"):
            raise TopologyError(f"bad kind for {nid!r}")
        parent = nd.get("parent")
        if parent is not None and not isinstance(parent, str):
            raise TopologyError("parent must be a string or null")
        up = nd.get("uplink")
        if up is not None:
            if not isinstance(up, dict) or set(up) != UPLINK_KEYS:
                raise TopologyError(f"uplink of {nid!r} needs exactly {sorted(UPLINK_KEYS)}")
            wt = up["w_t"]
            if isinstance(wt, bool) or not isinstance(wt, int) or wt < 1:
                raise TopologyError("w_t must be an integer >= 1")
            up = {"alpha": _num(up["alpha"], "alpha"), "beta": _num(up["beta"], "beta"),
                  "epsilon": _num(up["epsilon"], "epsilon"), "w_t": wt}
            if up["alpha"] < 0 or up["beta"] <= 0 or up["epsilon"] < 0:
                raise TopologyError("need alpha >= 0, beta > 0, epsilon >= 0")
        comp = nd.get("compute")
        if comp is not None:
            if not isinstance(comp, dict) or set(comp) != COMPUTE_KEYS:
                raise TopologyError(f"compute of {nid!r} needs exactly {sorted(COMPUTE_KEYS)}")
            comp = {"gamma": _num(comp["gamma"], "gamma"), "delta": _num(comp["delta"], "delta")}
            if comp["gamma"] < 0 or comp["delta"] < 0:
                raise TopologyError("need gamma, delta >= 0")
        nodes[nid] = Node(nid, kind, parent, up, comp)
    roots = [n.id for n in nodes.values() if n.parent is None]
    if len(roots) != 1:
        raise TopologyError(f"need exactly one root, found {len(roots)}")
    for n in nodes.values():
        if n.parent is not None:
            if n.parent not in nodes:
                raise TopologyError(f"parent {n.parent!r} of {n.id!r} does not exist")
            nodes[n.parent].children.append(n.id)
            if n.uplink is None:
                raise TopologyError(f"non-root {n.id!r} needs an uplink")
        elif n.uplink is not None:
            raise TopologyError("root must not have an uplink")
    # reachability from the root (detects cycles: a cycle is unreachable from the root)
    seen, stack = set(), [roots[0]]
    while stack:
        x = stack.pop()
        if x in seen:
            raise TopologyError("cycle")
        seen.add(x)
        stack.extend(nodes[x].children)
    if len(seen) != len(nodes):
        raise TopologyError("cycle or disconnected node")
    for n in nodes.values():
        if n.kind == "server":
            if n.children:
                raise TopologyError(f"server {n.id!r} has children")
            if n.compute is None:
                raise TopologyError(f"server {n.id!r} needs compute params")
        else:
            if not n.children:
                raise TopologyError(f"switch {n.id!r} is a leaf")
            if n.compute is not None:
                raise TopologyError(f"switch {n.id!r} must not have compute params")
    topo = Topology(nodes, roots[0], [], {})
    topo.servers = topo.servers_under(roots[0])
    if len(topo.servers) < 2:
        raise TopologyError("fewer than 2 servers")
    topo.rank = {s: i for i, s in enumerate(topo.servers)}
    return topo


# ---- document builders used by tests / configs (plain JSON, no method arithmetic) ----------

TABLE5 = {  # P:1080-1087, per float
    "cross_dc": {"alpha": 3.00e-2, "beta": 6.40e-9, "epsilon": 6.00e-11, "w_t": 9},
    "root_sw": {"alpha": 6.58e-3, "beta": 6.40e-10, "epsilon": 6.00e-12, "w_t": 9},
    "middle_sw": {"alpha": 6.58e-3, "beta": 6.40e-9, "epsilon": 1.22e-10, "w_t": 9},
    "server": {"gamma": 6.00e-10, "delta": 1.87e-10},
}


def single_switch_doc(n: int, link: dict, compute: dict) -> str:
    nodes = [{"id": "sw", "kind": "switch", "parent": None, "uplink": None}]
    for i in range(n):
        nodes.append({"id": f"s{i}", "kind": "server", "parent": "sw",
                      "uplink": dict(link), "compute": dict(compute)})
    return json.dumps({"nodes": nodes})


def two_level_doc(groups: list, mid_link: dict, leaf_link: dict, compute: dict) -> str:
    """Root -> len(groups) middle switches -> groups[g] servers each."""
    nodes = [{"id": "R", "kind": "switch", "parent": None, "uplink": None}]
    k = 0
    for g, cnt in enumerate(groups):
        nodes.append({"id": f"M{g}", "kind": "switch", "parent": "R", "uplink": dict(mid_link)})
        for _ in range(cnt):
            nodes.append({"id": f"s{k}", "kind": "server", "parent": f"M{g}",
                          "uplink": dict(leaf_link), "compute": dict(compute)})
            k += 1
    return json.dumps({"nodes": nodes})
