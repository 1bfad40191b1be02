# SM-partition A/B of the H-LU sweep (dev tool): one process per partition size
# (green contexts are made once per handle).  usage: bash tools/ab_green.sh c4 "0 96 112 120"
cfg=${1:-c4}
for rep in 1 2; do
  for n in ${2:-0 96 104 112 120 128}; do
    FDE_H2_GREEN=$n timeout 300 python tools/ab_inproc.py $cfg "FDE_H2_GREEN=$n" 2>&1 | grep "\[" | sed "s/^/rep=$rep /"
  done
done
