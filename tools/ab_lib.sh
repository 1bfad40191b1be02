# A/B of compile-time variants (dev tool): hlu period and factor time per library
for v in "" ${VARIANTS}; do
  lib=paper_1808_02937_b200/libfde.so; [ -n "$v" ] && lib=paper_1808_02937_b200/variants/libfde_$v.so
  for rep in 1 2; do
    p=$(FDE_LIB_PATH=$lib FDE_H2_HOLD_US=40000 FDE_DEBUG_TIMELINE=1 python tools/hlu_only.py 64 ${CFG:-c4} 2>&1 | grep "per-step" | tail -1 | sed 's/.*copies end \([0-9.]*\).*/\1/')
    f=$(FDE_LIB_PATH=$lib python tools/hlu_only.py 64 ${CFG:-c4} 2>&1 | tail -1 | awk '{print $3}')
    echo "lib=${v:-base} rep=$rep period_us=$p factor_ms=$f"
  done
done
