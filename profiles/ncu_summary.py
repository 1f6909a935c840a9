"""Summarise an ncu --set full report: per-kernel table + top source lines.

    python profiles/ncu_summary.py gpurun_out/X.ncu-rep [kernel-regex-for-source]
"""
import csv
import io
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[0], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    cols = [("dur_ms", "gpu__time_duration.sum"), ("dram_rd_GB", "dram__bytes_read.sum"),
            ("dram_wr_GB", "dram__bytes_write.sum"), ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            ("warps_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
            ("inst_Mwarp", "smsp__inst_executed.sum"), ("regs", "launch__registers_per_thread"),
            ("l2_Msect", "lts__t_sectors.sum")]
    print("| kernel | " + " | ".join(c for c, _ in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for d in data:
        name = d[idx["Kernel Name"]].split("(")[0].replace("pcb::<unnamed>::", "").replace("void ", "")
        vals = []
        for c, k in cols:
            v = d[idx[k]] if k in idx else ""
            try:
                f = float(v)
                if c == "inst_Mwarp" or c == "l2_Msect":
                    f /= 1e6
                vals.append(f"{f:.3f}" if f < 100 else f"{f:.0f}")
            except ValueError:
                vals.append(v)
        print(f"| {name} | " + " | ".join(vals) + " |")


def source(rep, kre, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr, acc = None, None, []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0] not in ("", "Function Name") and len(r) > 6:
            try:
                acc.append((int(r[4]), cur, r[0], r[1][:100], r))
            except ValueError:
                pass
    tot = sum(a[0] for a in acc) or 1
    idx = {h: i for i, h in enumerate(hdr or [])}
    stalls = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
    for samp, f, ln, src, r in sorted(acc, reverse=True)[:top]:
        st = sorted(((int(r[idx[s]]) if r[idx[s]].isdigit() else 0, s) for s in stalls), reverse=True)[:3]
        print(f"{samp * 100 / tot:5.1f}% {f}:{ln} {src} | " + ", ".join(f"{s[6:]} {v}" for v, s in st))


if __name__ == "__main__":
    raw(sys.argv[1])
    if len(sys.argv) > 2:
        source(sys.argv[1], sys.argv[2])
