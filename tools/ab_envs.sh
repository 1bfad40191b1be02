# factor time of the c4 / c5 H-LU under several environment settings (dev tool)
# usage: CFG=c4 bash tools/ab_envs.sh "ENV1=a ENV2=b" "ENV3=c" ...
for rep in 1 2; do
  for e in "$@"; do
    f=$(env $e python tools/hlu_only.py 64 ${CFG:-c4} 2>&1 | tail -1 | awk '{print $3}')
    echo "[$e] rep=$rep factor_ms=$f"
  done
done
