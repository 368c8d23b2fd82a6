"""Print the kernels of a torch.profiler chrome trace from the first potrf panel on (non-panel kernels)."""
import json
import sys

ev = [e for e in json.load(open(sys.argv[1]))["traceEvents"] if e.get("cat") in ("kernel",)]
ev.sort(key=lambda e: e["ts"])
t0 = [e for e in ev if "potrf_panel" in e["name"]][0]["ts"]
skip = set(sys.argv[2:]) if len(sys.argv) > 2 else {"15"}
for e in ev:
    if e["ts"] < t0 - 200 or "potrf_panel" in e["name"]:
        continue
    st = str(e["args"].get("stream"))
    if st in skip:
        continue
    nm = e["name"].replace("dlab::(anonymous namespace)::", "").replace("void ", "")[:80]
    print(f"{e['ts'] - t0:9.1f} +{e['dur']:8.1f} s{st} {nm} grid {e['args'].get('grid')}")
