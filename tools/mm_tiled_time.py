"""Time the tiled vs flat mat-mat on the BASELINE configs (graph-replayed, rotating copies)."""
import sys, json, time
import numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1805_10692_b200 as cd
from paper_1805_10692_b200 import synth
from paper_1805_10692_b200._native import force_path
import bench

res = {}
for name, b in [("alexnet-fc6", 64), ("vgg-fc6", 128), ("resnet-conv", 1568), ("large", 256)]:
    cfg = synth.config(name)
    if name == "large":
        wt = synth.make_weights_device(cfg, 0, torch.device("cuda"))
    else:
        wt = torch.from_numpy(synth.make_layer(cfg)[0]).cuda()
    x = synth.make_inputs(cfg, np.random.default_rng(1), b)
    for kind, enc_fn in (("cer", cd.encode_cer),):
        enc = enc_fn(wt)
        rot = 2 if name == "large" else 4
        copies = [bench._clone(cd, enc) for _ in range(rot)]
        xs = [torch.from_numpy(x).cuda() for _ in range(rot)]
        ys = [torch.empty((cfg.m, b), device="cuda") for _ in range(rot)]
        for path in ("flat", "tiled", "tiled_frag"):
            with force_path("matmat", path):
                t0 = time.time()
                for i in range(rot):
                    cd.dot_device(copies[i], xs[i], out=ys[i])
                torch.cuda.synchronize()
                first = time.time() - t0
                steps = 3 if name == "large" else 20
                secs = bench._graph_time(lambda i: cd.dot_device(copies[i], xs[i], out=ys[i]), steps, 3, rot, torch)
                res[f"{name}/{b}/{kind}/{path}"] = round(secs / steps * 1e6, 2)
                print(name, b, kind, path, "us", round(secs / steps * 1e6, 2), "first(s)", round(first, 3), flush=True)
        del copies, xs, ys, enc
    del wt
    torch.cuda.empty_cache()
print(json.dumps(res))
