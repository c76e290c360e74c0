"""Where the host-buffer (e2e) path spends its time: public API vs the bare C call vs its CUDA pieces."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_10692_b200 as cd  # noqa: E402
from paper_1805_10692_b200 import _native, kernels, synth  # noqa: E402


def per_call(fn, reps=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e6 / reps


def main():
    cfg = synth.config("alexnet-fc6")
    rng = np.random.default_rng(0)
    w = torch.from_numpy(synth.make_weights(cfg, rng)).cuda()
    x = synth.make_inputs(cfg, rng, 1).reshape(-1)
    enc = cd.encode_cer(w)
    out = {}
    out["public_dot_us"] = per_call(lambda: cd.dot(enc, x))
    enc_s = cd.encode_cser(w)
    out["public_dot_cser_us"] = per_call(lambda: cd.dot(enc_s, x))
    out["public_step_us"] = per_call(lambda: (cd.dot(enc, x), cd.dot(enc_s, x)))
    dev = enc.device_encoding()
    st = dev.struct()
    L = _native.lib()
    ws_bytes = L.cerdot_dot_host_workspace_bytes(st, 1)
    px, px_np, py, py_np, ws = kernels._IO.get(cfg.m, cfg.n, 1, ws_bytes)
    stream = torch.cuda.current_stream().cuda_stream
    args = (st, px.data_ptr(), 1, 1, py.data_ptr(), 1, ws.data_ptr(), ws.numel(), stream)
    out["c_dot_host_us"] = per_call(lambda: L.cerdot_dot_host(*args))
    out["copyto_astype_us"] = per_call(lambda: (np.copyto(px_np, x, casting="unsafe"), py_np.astype(np.float64)))
    out["current_stream_us"] = per_call(lambda: torch.cuda.current_stream().cuda_stream)
    dx = torch.empty(cfg.n, device="cuda")
    dy = torch.empty(cfg.m, device="cuda")
    s = torch.cuda.current_stream()
    out["h2d_sync_us"] = per_call(lambda: (dx.copy_(px, non_blocking=True), s.synchronize()))
    out["d2h_sync_us"] = per_call(lambda: (py.copy_(dy, non_blocking=True), s.synchronize()))
    out["kernel_sync_us"] = per_call(lambda: (cd.dot_device(enc, dx, out=dy), s.synchronize()))
    out["sync_only_us"] = per_call(lambda: s.synchronize())
    print(out)


if __name__ == "__main__":
    main()
