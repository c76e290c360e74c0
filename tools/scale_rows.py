import sys, os, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1805_10692_b200 as cd
from paper_1805_10692_b200 import synth, shard
from paper_1805_10692_b200._native import lib
cfg = synth.config("alexnet-fc6")
w, xs = synth.make_layer(cfg)
enc = cd.encode_cer(torch.from_numpy(w).cuda())
x = torch.from_numpy(xs[1]).cuda()
for path in ("1", "2"):
    lib().cerdot_set_kernel_path(0, int(path))  # CERDOT_PATH_MATVEC
    for rows in (512, 1024, 2048, 4096):
        e = shard.slice_rows(enc, 0, rows) if rows < 4096 else enc
        y = torch.empty(rows, device="cuda")
        for _ in range(5): cd.dot_device(e, x, out=y)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20): cd.dot_device(e, x, out=y)
        g.replay(); torch.cuda.synchronize()
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): g.replay()
        t.record(); torch.cuda.synchronize()
        print(json.dumps({"path": path, "rows": rows, "us": s.elapsed_time(t) * 1e3 / 200}))
