# Sensitivity of the c4 H-LU step period to each launch class (dev tool): a 20 us
# spin behind every launch of one class (FDE_H2_DELAY, results intact), device held
# until the host has enqueued everything; d(period)/20 us ~ 1 on the binding chain
cfg=${1:-c4}
for c in none ${CLASSES:-l i n d p g s x r t o c}; do
  v=$(FDE_H2_DELAY=$c:${DUS:-20} FDE_H2_HOLD_US=${HOLD:-40000} FDE_DEBUG_TIMELINE=1 python tools/hlu_only.py 64 $cfg 2>&1 | grep "per-step" | tail -1 | sed 's/.*LU(k+1) end \([0-9.]*\).*copies end \([0-9.]*\).*/\1 \2/')
  echo "delay=$c period(LU,copies)= $v"
done
