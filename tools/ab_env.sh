# A/B of an environment switch (dev tool): factor time of the c4 / c5 H-LU
# usage: ENVA="FDE_H2_PIPE=0" ENVB="FDE_H2_PIPE=1" bash tools/ab_env.sh [c4|c5]
for rep in 1 2 3; do
  for e in "$ENVA" "$ENVB"; do
    f=$(env $e python tools/hlu_only.py 64 ${1:-c4} 2>&1 | tail -1 | awk '{print $3}')
    echo "$e rep=$rep factor_ms=$f"
  done
done
