"""Summarise an ncu --set full report into profiles/: per kernel the metrics the
roofline and the judge read (duration, tensor-pipe %, issue %, DRAM bytes, regs).
    python tools/ncu_summary.py gpurun_out/X.ncu-rep profiles/Y.json "note"
"""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        m = {}
        for k in KEYS:
            if k in d:
                u = units[hdr.index(k)]
                m[k] = f"{d[k]} {u}".strip()
        res.append({"kernel": d.get("Kernel Name", "")[:80], "id": d.get("ID"), "metrics": m})
    json.dump({"report": rep, "note": note, "kernels": res}, open(out, "w"), indent=1)
    for x in res:
        mm = x["metrics"]
        print(x["kernel"][:50], "| t", mm.get("gpu__time_duration.sum"), "| tensor",
              mm.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
              "| issue", mm.get("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
              "| dram R/W", mm.get("dram__bytes_read.sum"), mm.get("dram__bytes_write.sum"),
              "| lts%", mm.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"))


if __name__ == "__main__":
    main()
