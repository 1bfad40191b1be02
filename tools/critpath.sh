# critical-path analysis of the c4 H-LU sweep (dev tool): device period per step with
# launch classes left out (FDE_H2_SKIP, results garbage) and the host held back
cfg=${1:-c4}
for sk in ${SKIPS:-none r x l i n lin d t o c g p s tgc}; do
  v=$(FDE_H2_SKIP=$sk FDE_H2_HOLD_US=${HOLD:-40000} FDE_DEBUG_TIMELINE=1 python tools/hlu_only.py 64 $cfg 2>&1 | grep "per-step" | tail -1 | sed 's/.*LU(k+1) end \([0-9.]*\).*copies end \([0-9.]*\).*/\1 \2/')
  echo "skip=$sk period(LU,copies)= $v"
done
