"""One encode call per kind of a config (for ncu): python tools/enc_one.py config [kind]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_10692_b200 as cd  # noqa: E402
from paper_1805_10692_b200 import synth  # noqa: E402

cfg = synth.config(sys.argv[1])
w = synth.make_weights_device(cfg, 0, "cuda")
kinds = sys.argv[2:] or ["cer"]
for kind in kinds:
    (cd.encode_cer if kind == "cer" else cd.encode_cser)(w)
torch.cuda.synchronize()
print("ok")
