"""Hash of the assembled dense operator (bit-level comparison of assembly paths) and
the assembly time -- dev tool.  usage: expand_hash.py c2|c3|c4|c5"""
import hashlib
import sys
import time
sys.path.insert(0, '.')
import torch  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402

cfg = sys.argv[1]
p = {"c2": lambda: fi.config2(1.5), "c3": lambda: fi.config3(16), "c4": fi.config4, "c5": lambda: fi.config5(nrhs=1)}[cfg]()
h = fde.Handle(0)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    op = fde.assemble_problem(h, p)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    A = fde.operator_dense_paper(h, op)
    hsh = hashlib.sha1(A.cpu().numpy().tobytes()).hexdigest()[:16]
    print(cfg, "assemble wall ms", round(1e3 * (t1 - t0), 2), "hash", hsh, flush=True)
    del A
    op.free()
