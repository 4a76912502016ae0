"""Generate planner/schedule golden vectors from the UNMODIFIED reference.

TEST INFRASTRUCTURE ONLY.  Run in the dev container, where the reference is
mounted read-only at /root/reference; the outputs are committed under
tests/golden/ so the parity tests run anywhere (the GPU box has no
/root/reference).

    python oracle/gen_golden.py            # rewrites tests/golden/planner_golden.json

For every case it records the reference's own outputs:
  * plan_json(plan(g, cfg)) (or the InfeasibleModelError message),
  * report_json and the sha256 of trace_to_csv of simulate() for m in {1, l, 4l},
  * compute_balanced / memory_balanced_* / split_pair on the graph.
Graphs are stored as reference profile documents (profile_doc).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
from pathlib import Path

REF = Path(os.environ.get("DAWNPLAN_REF", "/root/reference/pkg/src"))
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "planner_golden.json.gz"

MIB = 1 << 20
GIB = 1 << 30


def main() -> None:
    sys.path.insert(0, str(REF))
    import numpy as np
    import dawnplan as R
    import importlib
    sim_mod = importlib.import_module("dawnplan.simulate")

    graphs = []
    data = REF.parent / "tests" / "data"
    graphs.append(R.load_profile(data / "uni8.json"))
    graphs.append(R.load_profile(data / "tri4.json"))
    graphs.append(R.gen_uniform(8, 1000, MIB))
    for seed in (1, 2, 3):
        graphs.append(R.gen_transformer_like(2 + seed, seed))
        graphs.append(R.gen_cnn_like(4 + 4 * seed, seed))
    graphs.append(R.gen_cnn_like(16, 7))
    rng = np.random.default_rng(5150)
    for k in range(6):  # random chains in the regime of the reference acceptance tests
        n = int(rng.integers(12, 25))
        nodes = []
        for i in range(n):
            t = int(rng.integers(500, 1501))
            m = int(rng.integers(int(0.9 * MIB), int(1.1 * MIB) + 1))
            nid = f"n{i}"
            nodes.append(R.ProfiledNode(
                id=nid, depth=i, fwd_start=i, t_f=t // 2, t_b=t - t // 2, m_a=m, m_p=0, m_d=0,
                saved=(R.TensorRef(f"{nid}.a", m, nid, i),),
                consumers=(f"n{i + 1}",) if i + 1 < n else ()))
        graphs.append(R.ComputationGraph.build(f"chain{k}_{n}", nodes))

    cases = []
    for g in graphs:
        entry = {"profile": R.profile_doc(g), "hash": R.canonical_hash(g), "balance": [], "plans": []}
        n = len(g)
        for stages in (2, 3, 4, 8):
            if stages > n:
                continue
            cb = R.compute_balanced(g, 0, n - 1, [1] * stages)
            bal = {"stages": stages, "compute_balanced": list(cb.positions)}
            for name, fn in (("mem_1f1b", R.memory_balanced_1f1b), ("mem_sync", R.memory_balanced_sync)):
                try:
                    bal[name] = list(fn(g, stages).positions)
                except R.InfeasibleCutError as e:
                    bal[name] = "ERR:" + str(e)
            bal["split_pair"] = list(R.split_pair(g, 0, n - 1, stages, R.SCHEDULE_ASYNC,
                                                  list(range(1, stages // 2 + 1)),
                                                  list(range(stages // 2 + 1, stages + 1))))
            entry["balance"].append(bal)
            for sched in (R.SCHEDULE_ASYNC, R.SCHEDULE_SYNC):
                profs = R.stage_profiles(g, cb, stages, sched)
                top = max(p.sched_peak for p in profs)
                for frac in (2.0, 0.95, 0.6, 0.3):
                    for bw in (16 * GIB, 100 * MIB):
                        cap = max(1, int(frac * top))
                        cfg = R.PlanConfig(stages=stages, schedule=sched, capacity=cap, bandwidth=bw)
                        rec = {"stages": stages, "schedule": sched, "capacity": cap, "bandwidth": bw}
                        try:
                            p, trace = R.plan_with_trace(g, cfg)
                        except R.InfeasibleModelError as e:
                            rec["error"] = str(e)
                            entry["plans"].append(rec)
                            continue
                        pj = R.plan_json(p)
                        rec["plan_doc"] = json.loads(pj)
                        rec["plan_json_sha256"] = hashlib.sha256(pj.encode()).hexdigest()
                        rec["trace"] = [[s.lo, s.hi, s.first_stage, s.last_stage, s.cb, s.mb, s.chosen]
                                        for s in trace]
                        rec["sim"] = []
                        for m in sorted({1, stages, 4 * stages}):
                            r = R.simulate(p, g, R.SimConfig(micro_batches=m, schedule=sched,
                                                             bandwidth=bw, capacity=cap))
                            rec["sim"].append({"m": m, "report": json.loads(sim_mod.report_json(r)),
                                               "report_sha256": hashlib.sha256(sim_mod.report_json(r).encode()).hexdigest(),
                                               "csv_sha256": hashlib.sha256(R.trace_to_csv(r).encode()).hexdigest()})
                        entry["plans"].append(rec)
        cases.append(entry)
    OUT.parent.mkdir(parents=True, exist_ok=True)
    OUT.write_bytes(gzip.compress(json.dumps({"generator": "oracle/gen_golden.py", "reference": "dawnplan 0.1.0",
                               "cases": cases}, sort_keys=True).encode(), mtime=0))
    print(f"wrote {OUT} ({OUT.stat().st_size // 1024} KiB, {len(cases)} graphs)")


if __name__ == "__main__":
    main()
