"""Aggregate per-instruction warp-stall samples of one kernel from an ncu report.
    python tools/ncu_stalls.py REP KERNEL_REGEX [top]"""
import csv, io, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + rx,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = raw.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
S = h.index("Warp Stall Sampling (All Samples)")
st = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = {h[i]: 0 for i in st}
items = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    try:
        s = float(r[S] or 0)
    except ValueError:
        continue
    for i in st:
        try:
            tot[h[i]] += float(r[i] or 0)
        except ValueError:
            pass
    dom = max(st, key=lambda i: float(r[i] or 0) if r[i] not in ("", None) else 0)
    items.append((s, r[0], r[1], h[dom]))
T = sum(tot.values()) or 1
print("total samples", T)
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"  {k:28s} {100*v/T:5.1f}%")
print("top instructions:")
for s, a, src, d in sorted(items, reverse=True)[:top]:
    print(f"  {100*s/T:5.1f}% {a} {src[:70]:70s} {d}")
