"""Critical-chain view of a tiles_trace CSV (tools/peaks/tiles_trace.cu)."""
import csv
import sys

rows = list(csv.DictReader(open(sys.argv[1])))
T = {(int(r["i"]), int(r["j"])): r for r in rows}
nt = max(int(r["j"]) for r in rows) + 1
print("end", max(float(r["end_us"]) for r in rows))
js = list(range(0, min(nt, 6))) + list(range(6, nt, max(1, nt // 8)))
for j in js:
    d = T[(j, j)]
    s = T.get((j + 1, j))
    f = lambda r, k: float(r[k]) if r else 0.0
    print(f"j={j:2d} diag grab {f(d,'grab_us'):8.1f} upd {f(d,'update_us'):8.1f} end {f(d,'end_us'):8.1f} | "
          f"(j+1,j) grab {f(s,'grab_us'):8.1f} upd {f(s,'update_us'):8.1f} end {f(s,'end_us'):8.1f}")
