"""Print per-CTA phase timestamps of the window mat-vec (CERDOT_PATH_TRACE), relative to the earliest start.

Usage: python tools/trace_matvec.py [config:rows:kind ...]   (default alexnet-fc6:4096:cer/cser)
Needs a library built with -DCERDOT_TRACE_KERNELS (NVCC_EXTRA=-DCERDOT_TRACE_KERNELS python -m paper_1805_10692_b200.build --force).
"""
import os, re, subprocess, sys
code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1805_10692_b200 as cd
from paper_1805_10692_b200 import synth, shard
cfg = synth.config(sys.argv[1]); rows = int(sys.argv[2])
w, xs = synth.make_layer(cfg)
enc = (cd.encode_cser if sys.argv[3] == "cser" else cd.encode_cer)(torch.from_numpy(w).cuda())
e = shard.slice_rows(enc, 0, rows) if rows < cfg.m else enc
x = torch.from_numpy(xs[1]).cuda(); y = torch.empty(rows, device="cuda")
for _ in range(3): cd.dot_device(e, x, out=y)
torch.cuda.synchronize()
from paper_1805_10692_b200._native import lib
lib().cerdot_set_kernel_path(0, 1)  # CERDOT_PATH_MATVEC: the window kernel
for _ in range(3): cd.dot_device(e, x, out=y)
torch.cuda.synchronize()
lib().cerdot_set_kernel_path(4, 1)  # CERDOT_PATH_TRACE
cd.dot_device(e, x, out=y); torch.cuda.synchronize()
'''
cases = [tuple(a.split(":")) for a in sys.argv[1:]] or [("alexnet-fc6", "4096", "cer"), ("alexnet-fc6", "4096", "cser")]
for cfgname, rows, kind in cases:
    env = dict(os.environ)
    out = subprocess.run([sys.executable, "-c", code, cfgname, str(rows), kind], capture_output=True, text=True,
                         env=env).stdout
    recs = [list(map(int, re.findall(r"(\d+)", l)[:12])) for l in out.splitlines() if l.startswith("TRACE")]
    if not recs:
        print(out); continue
    t0 = min(r[3] for r in recs)
    print(f"== {cfgname} rows={rows} {kind}: us since first CTA start: start / prologue / after-wait / x-staged / end / gather+scan done / segments done / row written / cp.async drained")
    for r in recs:
        print(f"cta {r[0]:3d} warp {r[1]:2d} rows {r[2]}: " + " ".join(f"{(v - t0) / 1e3:7.2f}" for v in r[3:12]))
