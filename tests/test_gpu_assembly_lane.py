"""The lane-per-pair assembly path (k_pairs_lane) reproduces the
warp-per-pair path bit for bit: the same quadrature points, weights, kernel values
and fma sequences for every single-cell far pair.  FDE_ASM_LANE is read once per
process, so each path runs in a subprocess; the operators are compared by a
SHA-256 of their bytes (mirrored graded mesh N = 256, P = 8: 32,896 pairs, over
the lane path's launch threshold; and P = 4)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, {root!r})
import torch
import fde_inputs as fi
from paper_1808_02937_b200 import fde
h = fde.Handle(0)
p = fi.config4(N=256, P={P})
op = fde.assemble_problem(h, p)
A = fde.operator_rows_internal(h, op)
torch.cuda.synchronize()
print(hashlib.sha256(A.cpu().numpy().tobytes()).hexdigest())
"""


def _sha(lane, P):
    env = dict(os.environ, FDE_ASM_LANE=str(lane))
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, P=P)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("P", [8, 4])
def test_lane_path_bitwise_equals_warp_path(P):
    assert _sha(1, P) == _sha(0, P)
