P=${1:-r02e}
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${P}_smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${P}_gputests.txt 2>&1
python bench.py > gpurun_out/${P}_bench_c2_default.json 2> gpurun_out/${P}_bench_c2_default.err
python bench.py --steps 20 --warmup 5 > gpurun_out/${P}_bench_c2_steps20.json 2> /dev/null
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${P}_bench_reference.json 2> /dev/null
for c in C1 C3 C4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/${P}_bench_$c.json 2>/dev/null; done
