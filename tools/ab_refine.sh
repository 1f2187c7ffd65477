# A/B of library variants on the refinement-window pipeline (tools/refine_rate.py)
for v in "$@"; do
  if [ "$v" = default ]; then unset RF_LIB_PATH; else export RF_LIB_PATH=paper_1905_02082_b200/_variants/lib$v.so; fi
  echo -n "$v: "; python tools/refine_rate.py | tail -1
done
