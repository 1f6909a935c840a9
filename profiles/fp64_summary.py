"""FP64 kernels by measured instruction counts: turns the CSV of

    ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,
        sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,
        smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,
        smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,dram__bytes_read.sum,
        dram__bytes_write.sum --clock-control none -k regex:"k_lik|k_var_point|k_sample|k_prepare" --csv
        python bench.py --n 100000000 --subsets 800 --steps 1 --warmup 1 --no-e2e --no-cpu

into profiles/r02_fp64_pipe.json (per kernel and family: DFMA+DADD+DMUL per point, FP64 instructions per
second, FP64-pipe busy %, thread instructions per point, DRAM bytes per point). bench.py reads it for
roofline.per_kernel[*].fp64_measured.

    python profiles/fp64_summary.py gpurun_out/X_fp64_metrics.csv profiles/r02_fp64_pipe.json
"""
import collections
import csv
import json
import re
import sys

FAM = {"0": "gaussian", "1": "frank", "2": "gumbel"}


def main(src, dst, points=1e8):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ix = {n: i for i, n in enumerate(h)}
    agg = collections.OrderedDict()
    for r in data:
        d = agg.setdefault(r[ix["ID"]], {"kernel": r[ix["Kernel Name"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    out = {}
    for d in agg.values():
        m = re.search(r"(k_\w+)<(\d)(?:, (\w+))?(?:, (\d))?", d["kernel"])
        kn, fam = m.group(1), FAM[m.group(2)]
        if kn == "k_lik":
            kn = "k_lik(fp64)" if (m.group(3) == "double2" and m.group(4) == "0") else "k_lik(fp32 warm-up)"
        t = d["gpu__time_duration.sum"] * 1e-9
        if t < 1e-4:  # the short follow-up pass over a few blocks
            continue
        fp = sum(d[f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum"] for o in ("dfma", "dadd", "dmul"))
        out.setdefault(kn, {})[fam] = {
            "ms_per_1e8": t * 1e3 * 1e8 / points, "fp64_instr_per_point": fp / points, "fp64_instr_per_s": fp / t,
            "sm__pipe_fp64_cycles_active_pct": d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
            "thread_instr_per_point": d["smsp__inst_executed.sum"] * 32 / points,
            "dram_bytes_per_point": (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / points}
    json.dump({"source": f"ncu --metrics ({src}): python bench.py --n 1e8 --subsets 800, B200, clock-control none",
               "note": "fp64_instr = DFMA+DADD+DMUL thread instructions executed (dynamic); peak 1.847e13 instr/s "
                       "(pcb_measure_fp64_peak DFMA loop)", "kernels": out}, open(dst, "w"), indent=1)
    for kn, v in out.items():
        for fam, e in v.items():
            print(kn, fam, {a: round(b, 3) for a, b in e.items()})


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
