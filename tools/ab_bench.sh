#!/bin/bash
# A/B the bench over alternative builds of libfde.so, interleaved (dev tool)
# usage: ab_bench.sh ROUNDS lib1.so lib2.so ...   (extra bench args via BENCH_ARGS)
rounds=$1; shift
cp paper_1808_02937_b200/libfde.so /tmp/libfde_orig.so
for r in $(seq 1 $rounds); do
  for f in "$@"; do
    cp "$f" paper_1808_02937_b200/libfde.so
    v=$(python bench.py --steps 10 --warmup 3 --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],2))")
    echo "$r $(basename $f): $v"
  done
done
cp /tmp/libfde_orig.so paper_1808_02937_b200/libfde.so
