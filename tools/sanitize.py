"""Small invocations of every kernel family for compute-sanitizer runs."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2507_16099_b200 import ops

M, N, K = 256, 384, 512
x, w, dy = synth.linear_inputs("c2", M, N, K, seed=0)
X, W, G = (torch.from_numpy(a).to(torch.bfloat16).cuda() for a in (x, w, dy))
for gran in ("tensor", "row", "col", "row_col"):
    ops.cast(X, "e4m3", gran, want_q=True, want_qt=True)
ops.cast(X, "e4m3", "mx32", want_q=True, want_qt=True)
for recipe in ("tensorwise", "rowwise", "rowwise_gw_hp", "mxfp8"):
    plan = ops.LinearPlan(M, N, K, recipe=recipe)
    saved = plan.new_saved()
    plan.forward(X, W, saved)
    plan.backward(G, saved, x=X)
    plan.forward(X, W, None)
torch.cuda.synchronize()
print("ok")
