#!/usr/bin/env python
"""Prints a one-line summary of a bench.py JSON line file: tools/bench_summary.py FILE [label]."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
label = sys.argv[2] if len(sys.argv) > 2 else d.get("config", {}).get("workload", "")
keys = {k: d.get(k) for k in ("value", "exact_probes_per_sentence", "exact_ms_share")}
print(label, {k: (round(v, 4) if isinstance(v, float) else v) for k, v in keys.items()},
      "clock", d.get("clocks", {}).get("sm_mhz"), "batch", d.get("config", {}).get("sentences_per_step_per_gpu"))
