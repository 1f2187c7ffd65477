for rep in 1 2; do
for v in 0 1; do
  echo -n "RF_PDL=$v: "
  RF_PDL=$v python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"
done
done
