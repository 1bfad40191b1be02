# Round-end evidence on one B200 (dev tool): GPU tests, bench lines for the four
# BASELINE configs and the reference arm, the ncu launch list of the c4 bench and
# --set full captures of the dominant kernels.  usage: bash tools/final_evidence.sh TAG
T=${1:-r2e}
O=gpurun_out
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/${T}_gputest.txt 2>&1; tail -3 $O/${T}_gputest.txt
for c in c4 c2 c3 c5; do
  s=20; w=5; [ $c = c5 ] && s=6 && w=3
  timeout 900 python bench.py --config $c --steps $s --warmup $w > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err; tail -c 300 $O/${T}_bench_$c.json; echo
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/${T}_bench_reference.json 2>&1; tail -c 300 $O/${T}_bench_reference.json; echo
timeout 900 python bench.py --impl reference --config c3 --steps 2 --warmup 1 > $O/${T}_bench_reference_c3.json 2>&1
FDE_LAUNCH_CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline" timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/${T}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_gemv_bulk -s 2 -c 1 -o $O/${T}_gemv python tools/gemv_only.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_dmma -s 2 -c 1 -o $O/${T}_gemm python tools/gemm_only.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_apply_pf -s 2 -c 1 -o $O/${T}_apply python tools/apply_only.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:k_h2_gemm<.int.64, .int.64" -s 41 -c 1 -o $O/${T}_h2gemm python tools/hlu_only.py 64 c4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_h2_lu_reg -s 20 -c 1 -o $O/${T}_lureg python tools/hlu_only.py 64 c4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_bcore -s 60 -c 1 -o $O/${T}_bcore python tools/hlu_only.py 64 c4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_pairs_kernel|k_pairs_lane|k_expand_tiles" -s 0 -c 2 -o $O/${T}_asm python tools/gemv_only.py > /dev/null 2>&1
FDE_LAUNCH_CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline" python tools/profile_summary.py $O/${T}_launches.csv $O/${T} $O/${T}_gemv.ncu-rep $O/${T}_gemm.ncu-rep $O/${T}_apply.ncu-rep $O/${T}_h2gemm.ncu-rep $O/${T}_lureg.ncu-rep $O/${T}_bcore.ncu-rep $O/${T}_asm.ncu-rep
rm -f $O/*.ncu-rep $O/${T}_launches.csv   # (the summaries above are what is kept; gpurun_out is capped at 64 MiB)
ls -la $O | tail -30
