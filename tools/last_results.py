"""Print the sweep JSON lines of the last gpurun call (tool)."""
import json
from pathlib import Path

d = json.loads((Path(__file__).resolve().parents[1] / "gpurun_out" / ".last_call.json").read_text())
for line in d.get("stdout_tail", "").splitlines():
    if line.startswith("{"):
        r = json.loads(line)
        if "median_ms" in r:
            print(r.get("config"), r.get("variant"), round(r["median_ms"], 4), r.get("parity"))
        else:
            print(line[:300])
    elif line.strip() and not line.startswith("[gpurun]"):
        print(line[:300])
