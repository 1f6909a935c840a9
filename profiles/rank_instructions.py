"""Rank kernel instruction slots per key by phase and source line, from an
ncu --set full --import-source on report (first k_rank_cluster launch).

    python profiles/rank_instructions.py REPORT.ncu-rep KEYS [RANK_CU]

KEYS = keys that launch ranked (points x 2). Slots per key = warp
instructions x 32 / KEYS. Phases are the source ranges between the
"// ---- N." markers of rank.cu (the kernel's section comments)."""
import csv
import io
import re
import subprocess
import sys


def main(rep, keys, rank_cu="paper_1609_05530_b200/csrc/rank.cu"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:k_rank_cluster", "-c", "1"], capture_output=True, text=True).stdout
    rows, fname, hdr = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            nh = len(r)
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:  # ncu does not escape quotes inside inline-asm source lines: count from the row's end
            off = len(r) - nh
            ins = float(r[hdr["Instructions Executed"] + off] or 0)
            stall = float(r[hdr["Warp Stall Sampling (All Samples)"] + off] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((fname, int(r[0]), r[1], ins, stall))
    src = open(rank_cu).read().splitlines()
    marks = [(i + 1, m.group(1)) for i, l in enumerate(src) if (m := re.search(r"// ---- (\d+\.[^(]*)", l))]
    k0 = next(i + 1 for i, l in enumerate(src) if "k_rank_cluster_t(const ClusterJob" in l)
    k1 = next(i + 1 for i, l in enumerate(src) if i + 1 > k0 and l.startswith("}"))
    tot_ins = sum(r[3] for r in rows)
    tot_st = sum(r[4] for r in rows) or 1.0
    phase = {}
    for f, ln, _, ins, st in rows:
        if f != rank_cu.split("/")[-1] or not k0 <= ln <= k1:
            name = "helpers inlined from other files / other functions (order_key, atomics, cluster barrier)"
        else:
            name = "setup"
            for mln, mname in marks:
                if k0 <= mln <= ln:
                    name = mname.strip().rstrip(".")
        a = phase.setdefault(name, [0.0, 0.0])
        a[0] += ins
        a[1] += st
    print(f"total: {tot_ins * 32 / keys:.1f} instruction slots per key, {int(tot_st)} stall samples\n")
    print("| phase (kernel section) | slots / key | share of stall samples |\n|---|---|---|")
    for name, (ins, st) in sorted(phase.items(), key=lambda kv: -kv[1][0]):
        print(f"| {name} | {ins * 32 / keys:.1f} | {100 * st / tot_st:.1f}% |")
    print("\n| source line | slots / key | stall % | code |\n|---|---|---|---|")
    for f, ln, code, ins, st in sorted(rows, key=lambda r: -r[3])[:30]:
        print(f"| {f}:{ln} | {ins * 32 / keys:.1f} | {100 * st / tot_st:.1f} | `{code.strip()[:80]}` |")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), *sys.argv[3:])
