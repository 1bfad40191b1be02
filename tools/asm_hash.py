"""Hash of the assembled c4 operator and the assembly time (dev tool: bitwise A/B of assembly changes)."""
import sys, hashlib
sys.path.insert(0, '.')
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
p = fi.config4() if (len(sys.argv) < 2 or sys.argv[1] == "c4") else fi.config3(16)
h = fde.Handle(0)
for _ in range(2):
    op = fde.assemble_problem(h, p)
    torch.cuda.synchronize()
    t = op.info.assemble_ms
    A = fde.operator_rows_internal(h, op)
    dig = hashlib.sha256(A.cpu().numpy().tobytes()).hexdigest()[:16]
    op.free()
print("assemble_ms", round(t, 3), "sha", dig)
