# A/B of library builds on one box: trajectory fingerprints, then alternating
# driver-setting bench runs. Usage: bash tools/ab_bench.sh <variant>... (the
# in-tree build is "new"; variants are _variants/lib<name>.so).
V="$@"
python tools/traj_hash.py > gpurun_out/ab_hash_new.txt 2>&1
for v in $V; do RF_LIB_PATH=paper_1905_02082_b200/_variants/lib$v.so python tools/traj_hash.py > gpurun_out/ab_hash_$v.txt 2>&1; done
for i in 1 2 3; do
  for v in $V new; do
    if [ $v = new ]; then L=; else L=paper_1905_02082_b200/_variants/lib$v.so; fi
    RF_LIB_PATH=$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], d["value"], d["e2e"]["value"])' $v >> gpurun_out/ab.txt
  done
done
