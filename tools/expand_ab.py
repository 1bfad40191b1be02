"""Dense-expansion A/B: assemble configs and save (or compare) the operators and the
assembly times -- dev tool.  usage: python tools/expand_ab.py out.npz [ref.npz]"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
h = fde.Handle(0)
res = {}
for name, p in (("c4", fi.config4()), ("c2", fi.config2(1.5)), ("c3", fi.config3(16)), ("c1", fi.config1()),
                ("odd", fi.config4(N=37 * 2, P=4))):
    ts = []
    for _ in range(5):
        op = fde.assemble_problem(h, p)
        ts.append(op.info.assemble_ms)
        if _ < 4:
            op.free()
    res[name] = fde.operator_dense_paper(h, op).cpu().numpy()
    op.free()
    print(f"{name}: assemble {np.median(ts[1:]):.3f} ms", flush=True)
np.savez(sys.argv[1], **res)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    for k in res:
        print(k, "bitwise equal" if np.array_equal(res[k], ref[k]) else
              f"max abs diff {np.abs(res[k] - ref[k]).max():.3e}")
