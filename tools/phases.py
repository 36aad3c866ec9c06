"""Print ms/step and the V/U spmm and select phases of a bench.py JSON line (file argument)."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["ms_per_step"], {k: v["ms_per_call"] for k, v in d["phases"].items() if "select" in k or "spmm" in k})
