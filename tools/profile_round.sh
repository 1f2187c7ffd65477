# Round-end evidence: launch list, one --set full capture per hot kernel (C2),
# k_fuse at C3 (bricks beyond L2), and text exports of every report into
# gpurun_out/ (copied to profiles/ afterwards). Each ncu pass runs only after
# the same command exited 0 without ncu.
set -x
P=${1:-r02}
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_bench_steps30.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_track --launch-skip 20 -c 1 -o gpurun_out/${P}_track python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_ncu_t.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fuse$|k_alloc|k_cull" --launch-skip 60 -c 3 -o gpurun_out/${P}_volume python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_ncu_v.log 2>&1
python bench.py --config C3 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_c3_steps30.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fuse$" --launch-skip 25 -c 1 -o gpurun_out/${P}_c3_fuse python bench.py --config C3 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${P}_ncu_c3.log 2>&1
for r in track volume c3_fuse; do
  [ -f gpurun_out/${P}_$r.ncu-rep ] && ncu -i gpurun_out/${P}_$r.ncu-rep --page details --csv > gpurun_out/${P}_${r}_details.csv 2>/dev/null
  [ -f gpurun_out/${P}_$r.ncu-rep ] && ncu -i gpurun_out/${P}_$r.ncu-rep --page raw --csv > gpurun_out/${P}_${r}_raw.csv 2>/dev/null
done
RF_TRACE_FILE=gpurun_out/${P}_trace.bin python bench.py --steps 40 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/${P}_trace.bin > gpurun_out/${P}_trace_summary.txt 2>&1
python tools/barrier_bench.py > gpurun_out/${P}_barrier_bench.txt 2>&1
ls -la gpurun_out | tail -30
