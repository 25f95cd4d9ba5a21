"""Print a one-line summary of a bench.py JSON line read from stdin (label = argv[1])."""
import json
import sys

GEMMS = ("ffn_gemm1", "ffn_gemm2", "wgrad_w2", "dgrad_dA", "wgrad_w1", "dgrad_dX")
lines = [l for l in sys.stdin.read().splitlines() if l.startswith("{")]
if not lines:
    print(sys.argv[1] if len(sys.argv) > 1 else "", "no JSON line")
    sys.exit(0)
j = json.loads(lines[-1])
lab = sys.argv[1] if len(sys.argv) > 1 else ""
ks = j.get("kernels", {})
mode = sys.argv[2] if len(sys.argv) > 2 else "gemm"
sel = {k: v["avg_ms"] for k, v in ks.items() if (mode == "all" or k in GEMMS)}
print(lab, j.get("ms_per_step"), (j.get("clocks") or {}).get("sm_mhz"), sel)
