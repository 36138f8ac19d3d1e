"""Prints the headline fields of bench.py JSON lines read from stdin (last line)."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
o = d.get("other_configs", {})
sl = d.get("serving_loop", {})
print("c2 step", round(d["us_per_step"], 2), "kernel", round(d["roofline"]["split_us"], 2),
      "e2e", round(d["e2e"]["ms_per_step"] * 1e3, 2) if "ms_per_step" in d.get("e2e", {}) else d.get("e2e"),
      "| loop step", round(sl.get("graph_step_us", 0), 1), "flush", round(sl.get("flush_step_us", 0), 1),
      "| " + " ".join(k.split("_")[0] + " " + str(round(x["us_per_step"], 1)) for k, x in o.items()
                      if isinstance(x, dict) and "us_per_step" in x))
