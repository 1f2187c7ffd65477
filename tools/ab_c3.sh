# A/B of k_fuse builds: C3 (k_fuse-heavy) and C2 bench lines, alternating.
V="$@"
for i in 1 2; do
  for v in $V new; do
    if [ $v = new ]; then L=; else L=paper_1905_02082_b200/_variants/lib$v.so; fi
    for c in C3 C2; do
      RF_LIB_PATH=$L python bench.py --config $c --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d.get("kernels") or {}; print(sys.argv[1], sys.argv[2], d["value"], d["e2e"]["value"])' $v $c >> gpurun_out/ab_c3.txt
    done
  done
done
