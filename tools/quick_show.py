"""Print the key numbers of gpurun_out/quick_*.log (tools/quick.sh)."""
import glob
import json

for f in sorted(glob.glob("gpurun_out/quick_[0-9]*.log")):
    txt = open(f).read()
    tag = [l for l in txt.splitlines() if l.startswith("# ")]
    L = [l for l in txt.splitlines() if l.startswith("{")]
    if not L:
        print(f, tag, txt[-800:])
        continue
    d = json.loads(L[0])
    ph = {k: round(v * 1e3, 1) for k, v in d.get("pcg_phases_ms_per_iteration", {}).items()}
    print(f, tag, "value", round(d["value"], 4), "ms/step", round(d["ms_per_step"], 3), "it_ms",
          round(d["pcg_iteration_roofline"]["ms_per_iteration"], 4), ph)
