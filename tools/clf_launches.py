#!/usr/bin/env python
"""Developer tool (under gpurun + ncu): one eager classifier forward at S=8192, B=1, so that
`ncu --metrics gpu__time_duration.sum` lists every kernel of the forward with its duration."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, init_weights  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cfg = ClassifierConfig()
clf = Classifier(cfg, init_weights(cfg, 7), torch.device("cuda:0"))
ids = torch.randint(0, cfg.vocab_size, (1, S), device="cuda")
mask = torch.ones(1, S, device="cuda")
mask[:, S - S // 8:] = 0
for _ in range(2):
    clf.forward(ids, mask)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured_forward")
clf.forward(ids, mask)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
