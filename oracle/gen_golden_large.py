"""Golden plans on the B200-measured BASELINE-model profiles, from the
UNMODIFIED reference.

TEST INFRASTRUCTURE ONLY.  Run in the dev container, where the reference is
mounted read-only at /root/reference:

    python oracle/gen_golden_large.py    # writes tests/golden/planner_golden_large.json.gz

Inputs are the schema-1 profiles measured on a B200 by
`python -m paper_2505_05856_b200 profile MODEL --micro-batch B` (committed as
tests/golden/profiles/*.json.gz): BERT-base b8 (111 nodes), BERT-large b32 /
b8 (219 nodes), GPT-2 XL b4 (435 nodes) and T5-large b16 (509 nodes).  For
each (profile, stages, capacity) case it records what the reference's own
`dawnplan.plan_with_trace` returns -- the plan_json bytes (sha256 + parsed
document) and the search trace, or the InfeasibleModelError message -- plus
`simulate` at m = 4l (report sha256 and document) and the reference's wall
time.  Capacities are fractions of the compute-balanced baseline's largest
sched_peak (memopt-active below 1.0) and the 40 GiB cap of BASELINE configs[2].
The reference needs minutes per GPT-2 XL / T5-large plan; expect ~40 min.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time
from pathlib import Path

REF = Path(os.environ.get("DAWNPLAN_REF", "/root/reference/pkg/src"))
HERE = Path(__file__).resolve().parent.parent / "tests" / "golden"
OUT = HERE / "planner_golden_large.json.gz"
GIB = 1 << 30

CASES = [
    # (profile, stages, capacity: float = fraction of the baseline's top sched_peak | int bytes)
    ("bert-base_b8", 4, 2.0),
    ("bert-base_b8", 4, 0.45),
    ("bert-large_b32", 8, 2.0),
    ("bert-large_b32", 8, 0.5),
    ("bert-large_b32", 8, 0.3),
    ("bert-large_b32", 4, 0.4),
    ("bert-large_b8", 8, 0.35),
    ("gpt2-xl_b4", 8, 40 * GIB),
    ("gpt2-xl_b4", 8, 0.5),
    ("gpt2-xl_b4", 4, 0.45),
    ("t5-large_b16", 8, 0.5),
    ("t5-large_b16", 4, 0.5),
]


def main() -> None:
    sys.path.insert(0, str(REF))
    import dawnplan as R
    sim_mod = __import__("dawnplan.simulate", fromlist=["report_json"])
    only = set(sys.argv[1:])
    old = {}
    if OUT.exists():
        for rec in json.loads(gzip.decompress(OUT.read_bytes()))["cases"]:
            old[(rec["profile"], rec["stages"], rec["capacity_spec"])] = rec
    out = []
    for name, stages, capspec in CASES:
        key = (name, stages, capspec)
        if only and name not in only and key in old:
            out.append(old[key])
            continue
        path = HERE / "profiles" / f"{name}.json.gz"
        tmp = Path("/tmp") / f"{name}.json"
        tmp.write_bytes(gzip.decompress(path.read_bytes()))
        g = R.load_profile(tmp)
        sched = R.SCHEDULE_ASYNC
        if isinstance(capspec, float):
            cb = R.compute_balanced(g, 0, len(g.nodes) - 1, [1] * stages)
            top = max(p.sched_peak for p in R.stage_profiles(g, cb, stages, sched))
            cap = int(capspec * top)
        else:
            cap = capspec
        bw = 16 * GIB
        rec = {"profile": name, "stages": stages, "capacity_spec": capspec, "capacity": cap,
               "bandwidth": bw, "schedule": sched, "hash": R.canonical_hash(g)}
        t0 = time.time()
        try:
            p, trace = R.plan_with_trace(g, R.PlanConfig(stages=stages, schedule=sched, capacity=cap,
                                                         bandwidth=bw))
        except R.InfeasibleModelError as e:
            rec["error"] = str(e)
        else:
            pj = R.plan_json(p)
            rec["plan_doc"] = json.loads(pj)
            rec["plan_json_sha256"] = hashlib.sha256(pj.encode()).hexdigest()
            rec["trace"] = [[s.lo, s.hi, s.first_stage, s.last_stage, s.cb, s.mb, s.chosen]
                            for s in trace]
            r = R.simulate(p, g, R.SimConfig(micro_batches=4 * stages, schedule=sched, bandwidth=bw,
                                             capacity=cap))
            rj = sim_mod.report_json(r)
            rec["sim"] = {"m": 4 * stages, "report_sha256": hashlib.sha256(rj.encode()).hexdigest(),
                          "iteration_time_us": json.loads(rj)["iteration_time_us"]}
        rec["reference_plan_s"] = round(time.time() - t0, 2)
        print(f"{name} l={stages} cap={cap}: {rec.get('error') or rec['plan_doc']['cuts']} "
              f"({rec['reference_plan_s']} s)", flush=True)
        out.append(rec)
        OUT.write_bytes(gzip.compress(json.dumps({"generator": "oracle/gen_golden_large.py",
                                                  "reference": "dawnplan 0.1.0", "cases": out},
                                                 sort_keys=True).encode(), mtime=0))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
