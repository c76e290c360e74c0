"""Summarise a tools/ncu_one.sh capture: headline sections, stall reasons, hottest SASS lines.
Usage: python tools/ncu_summary.py gpurun_out/TAG [n_hot]"""
import csv
import re
import sys

base = sys.argv[1]
nhot = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for line in open(base + ".details.txt"):
    if re.search(r"Duration|DRAM Through|L1/TEX Hit|L2 Hit|Issued Warp|Eligible Warps|Registers Per|Achieved Occ|"
                 r"L1/TEX Cache Through|Compute \(SM\)", line):
        print(line.rstrip())
rows = list(csv.reader(open(base + ".raw.csv")))
d = dict(zip(rows[0], rows[2]))
for k, v in d.items():
    if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            if float(v) > 0.1:
                print("  stall", k.replace("smsp__average_warps_issue_stalled_", "").replace(
                    "_per_issue_active.ratio", ""), v)
        except ValueError:
            pass
for k in ("smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__cycles_elapsed.avg"):
    print(" ", k, d.get(k))
rows = list(csv.reader(open(base + ".sass.csv")))
h = rows[1]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
for r in sorted(rows[2:], key=lambda r: -float(r[st] or 0))[:nhot]:
    print(f"{r[st]:>7} {r[ie]:>9}  {r[src].strip()}")
