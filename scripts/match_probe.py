#!/usr/bin/env python
"""Config-2 match timing alone: the request's plan run repeatedly with CUDA events around
the distance kernel (kvcomm_plan_set_match_events), results not checked (so probe builds
that skip work can be timed too).  Prints one JSON line.

  python scripts/match_probe.py [--steps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth
from synth.state import build_five_agent_state


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    w = synth.five_agent_workload()
    st = build_five_agent_state(w, seed=0, device=0, gamma=0.3)
    req = st.request
    plan = req.plan
    q = [st.queries[n] for n in req.names]
    for _ in range(3):
        plan.run(q)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for e in evs:
        plan.set_match_events(*e)
        plan.run(q)
    torch.cuda.synchronize()
    plan.set_match_events(None, None)
    ms = sorted(a.elapsed_time(b) for a, b in evs)
    nbytes = sum(st.queries[n].shape[0] * (w.capacity + 1) * st.queries[n].shape[1] * 2 for n in req.names)
    med = ms[len(ms) // 2]
    print(json.dumps({"match_ms_median": med, "match_ms_min": ms[0], "bytes": nbytes,
                      "GBps_median": nbytes / (med / 1e3) / 1e9, "lib": os.environ.get("KVCOMM_LIB", "in-tree")}))


if __name__ == "__main__":
    main()
