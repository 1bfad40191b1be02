"""Real (not extrapolated) timings of the CPU oracle on configs 2 and 3 -- the full
cold solve it performs: assembly of A (element-pair quadrature), load vector +
lifting, equilibrated LU with long-double refinement.  Median of 3, all host
cores and 1 thread.  usage: python tools/oracle_timing.py [out.jsonl]"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import fde_inputs as fi  # noqa: E402
import oracle as O  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else None
cores = os.cpu_count() or 1
thr_list = [int(sys.argv[2])] if len(sys.argv) > 2 else [cores]
for name, p in (("c2 (alpha 1.5)", fi.config2(1.5)), ("c3 (P=16)", fi.config3(16))):
    for threads in thr_list:
        reps = []
        for _ in range(3):
            t0 = time.perf_counter()
            sysm = O.assemble_system(p, threads=threads)
            t1 = time.perf_counter()
            G = np.stack([O.rhs(p, sysm, f) for f in p.forcings], axis=1)
            t2 = time.perf_counter()
            X = O.solve_dense(sysm.A, G)
            t3 = time.perf_counter()
            reps.append((t1 - t0, t2 - t1, t3 - t2, t3 - t0))
        med = [statistics.median(r[i] for r in reps) for i in range(4)]
        rec = {"config": name, "n": p.n, "threads": threads, "assemble_s": med[0], "rhs_s": med[1],
               "lu_refine_s": med[2], "total_s": med[3], "solves_per_s": len(p.forcings) / med[3],
               "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default"),
               "cpu": os.popen("lscpu | grep 'Model name'").read().strip()}
        print(json.dumps(rec), flush=True)
        if out:
            with open(out, "a") as f:
                f.write(json.dumps(rec) + "\n")
