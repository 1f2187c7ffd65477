set -x
python bench.py > gpurun_out/r01b_bench_default.log 2>&1
tail -1 gpurun_out/r01b_bench_default.log > gpurun_out/r01b_bench_default.json
python bench.py --impl reference > gpurun_out/r01b_bench_reference.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01b_launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track --launch-skip 20 -c 1 -o gpurun_out/r01b_track python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_t.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fuse|k_alloc|k_cull" --launch-skip 60 -c 3 -o gpurun_out/r01b_volume python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_v.log 2>&1
ls -la gpurun_out
