"""Regenerate profiles/ncu_traffic.json (bench.py's roofline.traffic) from an ncu capture of the CURRENT
library: DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of the headline CER and CSER
mat-vec kernels on the AlexNet-fc6 layer, each call cold (a fresh encoding copy per launch).

    python tools/ncu_traffic.py            (GPU box; runs ncu on itself with --child)
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def child():
    import numpy as np
    import torch

    sys.path.insert(0, ROOT)
    import bench
    import paper_1805_10692_b200 as cd
    from paper_1805_10692_b200 import synth

    cfg = synth.config("alexnet-fc6")
    w = torch.from_numpy(synth.make_weights(cfg, np.random.default_rng(0))).cuda()
    x = torch.from_numpy(synth.input_for(cfg, 0, 1)).cuda()
    for enc in (cd.encode_cer(w), cd.encode_cser(w)):
        for _ in range(3):  # three cold launches per kind (own arena copy each)
            cd.dot_device(bench._clone(cd, enc), x)
    torch.cuda.synchronize()


def main():
    if "--child" in sys.argv:
        return child()
    log = os.path.join(ROOT, "gpurun_out", "ncu_traffic.csv")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    subprocess.run(["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
                    "--clock-control", "none", "--cache-control", "all", "-k", "regex:k_matvec", "--csv",
                    "--log-file", log, sys.executable, os.path.abspath(__file__), "--child"], check=True)
    rows = [r for r in csv.reader(open(log)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launches = {}
    for r in rows[1:]:
        d = launches.setdefault(r[ii], {"kernel": r[ki]})
        v = float(r[vi].replace(",", ""))
        if r[mi].startswith("dram__bytes"):
            d["bytes"] = d.get("bytes", 0.0) + v * scale.get(r[ui], 1)
    per = [launches[k] for k in sorted(launches, key=int)]
    cer = [p["bytes"] for p in per[:3]]
    cser = [p["bytes"] for p in per[3:6]]
    out = {"_source": "tools/ncu_traffic.py: ncu --cache-control all, dram__bytes_read.sum + dram__bytes_write.sum "
                      "per launch of k_matvec (three cold launches each), library at the committed HEAD",
           "_kernels": sorted({p["kernel"][:80] for p in per}),
           "alexnet-fc6": {"cer": int(sum(cer) / len(cer)), "cser": int(sum(cser) / len(cser))}}
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
