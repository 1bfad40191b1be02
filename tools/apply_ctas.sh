# apply time vs cooperative grid size (dev tool)
for c in c2 c3 c4; do
  for n in 148 96 64 32 16; do
    echo "ctas=$n $(FDE_APPLY_CTAS=$n python tools/apply_only.py 1 $c 2>&1 | tail -1)"
  done
done
