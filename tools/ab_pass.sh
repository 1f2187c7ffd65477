# Per-pass A/B of library variants: bash tools/ab_pass.sh default name1 ...
for v in "$@"; do
  if [ "$v" = default ]; then unset RF_LIB_PATH; else export RF_LIB_PATH=paper_1905_02082_b200/_variants/lib$v.so; fi
  echo -n "$v: "; python tools/pass_bench.py 2>&1 | tail -1
done
