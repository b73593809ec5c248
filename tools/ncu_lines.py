"""Per-CUDA-source-line instruction counts and stall samples of one kernel.
    python tools/ncu_lines.py REP KERNEL_REGEX [top]"""
import csv, io, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + rx,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
agg = {}
fname = "?"
hdr = None
cur = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        iS = 4; iI = hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1][:60])
        continue
    try:
        s = float(r[iS] or 0); n = float(r[iI] or 0)
    except (ValueError, IndexError):
        continue
    a = agg.setdefault(cur, [0.0, 0.0])
    a[0] += s; a[1] += n
TS = sum(v[0] for v in agg.values()) or 1
TI = sum(v[1] for v in agg.values()) or 1
print(f"samples {TS:.0f} warp-instr {TI:.3e}")
print("by instructions executed:")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"  {100*v[1]/TI:5.1f}%I {100*v[0]/TS:5.1f}%S {k[0]}:{k[1]} {k[2]}")
print("by stall samples:")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"  {100*v[1]/TI:5.1f}%I {100*v[0]/TS:5.1f}%S {k[0]}:{k[1]} {k[2]}")
