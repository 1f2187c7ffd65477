# Round-end evidence: bench lines, ncu launch list, one --set full capture per hot kernel.
# Each ncu pass runs only after the same command exited 0 without ncu.
set -x
P=${1:-r01}
python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; tail -2 gpurun_out/${P}_pytest_gpu.log
python bench.py > gpurun_out/${P}_bench_default.log 2>&1 && tail -1 gpurun_out/${P}_bench_default.log > gpurun_out/${P}_bench_default.json
python bench.py --impl reference > gpurun_out/${P}_bench_reference.log 2>&1 && tail -1 gpurun_out/${P}_bench_reference.log > gpurun_out/${P}_bench_reference.json
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_bench_steps30.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track --launch-skip 20 -c 1 -o gpurun_out/${P}_track python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_ncu_t.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fuse|k_alloc|k_cull" --launch-skip 60 -c 3 -o gpurun_out/${P}_volume python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_ncu_v.log 2>&1
RF_TRACE_FILE=gpurun_out/${P}_trace.bin python bench.py --steps 40 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/${P}_trace.bin > gpurun_out/${P}_trace_summary.txt 2>&1
python tools/refine_rate.py > gpurun_out/${P}_refine_rate.txt 2>&1
python tools/config_rates.py > gpurun_out/${P}_config_rates.txt 2>&1
python tools/eval_rate.py > gpurun_out/${P}_eval_rate.txt 2>&1
ls -la gpurun_out
