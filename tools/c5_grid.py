"""C5 device-resident DFS rate vs the model kernel's grid size (ct_config.grid_override)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_18413_b200 import Model
from workloads.csp import csp_model

m = csp_model(30, 40, 12, 1_000_000, seed=7)
out = {}
ref = None
for g in [int(x) for x in (sys.argv[1:] or ["0", "96", "74", "48", "32"])]:
    M = Model(m["vlo"], m["vd"], m["scopes"], m["tables"], grid_override=g)
    M.search(value_order=0, max_nodes=200, max_solutions=0)
    t = time.perf_counter()
    st, sol, stats = M.search(value_order=0, max_nodes=3000, max_solutions=0, driver="device")
    dt = time.perf_counter() - t
    if ref is None:
        ref = (stats.nodes, stats.trace_hash)
    out[g] = {"us_per_node": dt / stats.nodes * 1e6, "same_trace": (stats.nodes, stats.trace_hash) == ref}
    M.close()
print(json.dumps(out))
