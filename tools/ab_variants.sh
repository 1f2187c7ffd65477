# A/B of library variants built with `python -m paper_1905_02082_b200.build --variant NAME -D...`
# usage: bash tools/ab_variants.sh name1 name2 ...   ("default" = the in-tree library)
# AB_ARGS overrides the bench arguments (unset: --steps 100 --warmup 5; AB_ARGS= : the default bench run)
for v in "$@"; do
  if [ "$v" = default ]; then unset RF_LIB_PATH; else export RF_LIB_PATH=paper_1905_02082_b200/_variants/lib$v.so; fi
  for rep in 1 2; do
    echo -n "$v: "
    python bench.py ${AB_ARGS---steps 100 --warmup 5} --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms_per_frame'])"
  done
done
