"""Kernel timing probe: eager vs graph, cold (rotating copies) vs warm, per config (GPU only)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1805_10692_b200 as cd  # noqa: E402
from paper_1805_10692_b200 import synth  # noqa: E402


def ev_time(fn, reps):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(reps):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="alexnet-fc6")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--kind", default="cer")
    args = ap.parse_args()
    cfg = synth.config(args.config)
    rng = np.random.default_rng(0)
    w = synth.make_weights(cfg, rng)
    x = synth.make_inputs(cfg, rng, args.batch)
    wt = torch.from_numpy(w).cuda()
    enc = (cd.encode_cer if args.kind == "cer" else cd.encode_cser)(wt)
    R = 16
    copies = [bench._clone(cd, enc) for _ in range(R)]
    xs = [torch.from_numpy(x).cuda() for _ in range(R)]
    ys = [torch.empty((cfg.m,) if args.batch == 1 else (cfg.m, args.batch), device="cuda") for _ in range(R)]
    out = {"config": cfg.name, "batch": args.batch, "kind": args.kind, "format_bytes": cd.storage_bits(enc) // 8}
    for i in range(5):
        cd.dot_device(enc, xs[0], out=ys[0])
    out["eager_warm_us"] = ev_time(lambda i: cd.dot_device(enc, xs[0], out=ys[0]), args.reps)
    out["eager_cold_us"] = ev_time(lambda i: cd.dot_device(copies[i % R], xs[i % R], out=ys[i % R]), args.reps)
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        cd.dot_device(copies[0], xs[0], out=ys[0])
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for i in range(R):
            cd.dot_device(copies[i], xs[i], out=ys[i])
    g.replay()
    torch.cuda.synchronize()
    out["graph_cold_us"] = ev_time(lambda i: g.replay(), max(1, args.reps // R)) / R
    # host launch cost
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.reps):
        cd.dot_device(enc, xs[0], out=ys[0])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    out["host_launch_us"] = (t1 - t0) * 1e6 / args.reps
    print(json.dumps(out))


if __name__ == "__main__":
    main()
