"""Topology documents used by several tests (plain JSON builders, no method arithmetic)."""
import json


def cross_dc(m0, c0, m1, c1, cross_eps=5e-9):
    """Two data centres joined by one slow, incast-prone link (w_t = 2) — small enough to run
    emulated on one GPU, and built so that GenTree adopts data rearrangement for
    the DC children of the top switch and ACPS above them."""
    nodes = [{"id": "X", "kind": "switch", "parent": None, "uplink": None}]
    k = 0
    for dc, (m, cnt) in enumerate([(m0, c0), (m1, c1)]):
        nodes.append({"id": f"DC{dc}", "kind": "switch", "parent": "X",
                      "uplink": {"alpha": 1e-3, "beta": 6.4e-9, "epsilon": cross_eps, "w_t": 2}})
        for g in range(m):
            nodes.append({"id": f"DC{dc}M{g}", "kind": "switch", "parent": f"DC{dc}",
                          "uplink": {"alpha": 1e-5, "beta": 6.4e-11, "epsilon": 0.0, "w_t": 9}})
            for _ in range(cnt):
                nodes.append({"id": f"s{k}", "kind": "server", "parent": f"DC{dc}M{g}",
                              "uplink": {"alpha": 1e-5, "beta": 6.4e-11, "epsilon": 0.0, "w_t": 9},
                              "compute": {"gamma": 6e-12, "delta": 1.87e-12}})
                k += 1
    return json.dumps({"nodes": nodes})
