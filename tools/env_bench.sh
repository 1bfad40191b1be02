#!/bin/bash
# bench c4 under alternative environment settings, interleaved (dev tool)
# usage: env_bench.sh ROUNDS "VAR=a" "VAR=b" ...   ("-" = no extra setting)
rounds=$1; shift
for r in $(seq 1 $rounds); do
  for e in "$@"; do
    if [ "$e" = "-" ]; then e=""; fi
    v=$(env $e python bench.py --steps 10 --warmup 3 --no-cpu-baseline $BENCH_ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],2))")
    echo "$r [$e]: $v"
  done
done
