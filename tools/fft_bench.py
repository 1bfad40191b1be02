"""Time the Toeplitz FFT stiffness matvec (uniform and single-ratio geometric meshes)
against the dense one and an empty-kernel launch floor -- measurement tool for
SURVEY 8(d) row a7 (latency-bound: 3 launches per pass, 2 passes on geometric
meshes, + the scatter).  usage: python tools/fft_bench.py"""
import sys
sys.path.insert(0, '.')
import torch  # noqa: E402
import fde_inputs as fi  # noqa: E402
from paper_1808_02937_b200 import fde  # noqa: E402


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / reps


stream = torch.cuda.current_stream()
h = fde.Handle(0, stream=stream.cuda_stream)
z = torch.zeros(1, device="cuda")
floor = timed(lambda: z.add_(0))
print(f"launch floor (one empty elementwise kernel): {floor:.1f} us")
cases = [("uniform c2 N=256 P=8", fi.config2(1.5)),
         ("geometric q=1.01 N=256 P=8", fi.geometric_problem(1.01, N=256, P=8)),
         ("uniform N=4096 P=8 (c5 mesh)", fi.config2(1.6, N=4096, P=8)),
         ("geometric q=1.001 N=4096 P=8", fi.geometric_problem(1.001, N=4096, P=8, alpha=1.6))]
for name, p in cases:
    op = fde.assemble_problem(h, p, flags=fde.OP_DENSE | fde.OP_TOEPLITZ)
    for nrhs in (1, 64):
        X = torch.randn(nrhs, p.n, dtype=torch.float64, device="cuda")
        tf = timed(lambda: fde.stiffness_matvec(h, op, X, path=fde.PATH_TOEPLITZ))
        td = timed(lambda: fde.stiffness_matvec(h, op, X, path=fde.PATH_DENSE))
        print(f"{name:32s} nrhs {nrhs:3d}: FFT {tf:8.1f} us  dense {td:8.1f} us  (FFT / launch floor {tf / floor:5.1f})")
    op.free()
