# Round profile captures of the current kernel (run under gpurun; every ncu
# command only after the same command exited 0 without ncu).  Outputs go to
# gpurun_out/; the summaries worth keeping are copied to profiles/rNN/.
set -x
python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b_pre.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/ncu_one.py --config kron27 --runs 16 > gpurun_out/one16.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bfs_persistent --csv --log-file gpurun_out/traffic16.csv python tools/ncu_one.py --config kron27 --runs 16 > gpurun_out/ncu_t16.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bfs_persistent -s 0 -c 1 -o gpurun_out/kron_full python tools/ncu_one.py --config kron27 --runs 1 > gpurun_out/ncu_full.log 2>&1
