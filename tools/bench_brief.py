"""Run bench.py (arguments passed through) and print the key numbers of its JSON line (dev helper)."""
import json
import subprocess
import sys
from pathlib import Path

root = Path(__file__).resolve().parents[1]
out = subprocess.run([sys.executable, str(root / "bench.py")] + sys.argv[1:], capture_output=True, text=True)
line = next((x for x in reversed(out.stdout.splitlines()) if x.startswith("{")), None)
if line is None:
    print(out.stdout[-2000:], out.stderr[-2000:])
    sys.exit(1)
d = json.loads(line)
r = d["roofline"]
print("ms/op", round(d["ms_per_step"], 4), "frac", round(r["frac"], 4), "op_frac", round(r["op_frac"], 4), "pass1/2",
      round(r["kernel_ms_pass1"], 4), round(r["kernel_ms_pass2"], 4), "fixups", round(r["fixup_ms_pass1"], 4),
      round(r["fixup_ms_pass2"], 4), "clocks", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
for k, v in d.get("secondary", {}).items():
    print(k, v.get("ms_per_op"), v.get("roofline_frac"), v.get("error"))
