set -x
python tools/ncu_one.py --config kron27 --runs 1 > gpurun_out/one.log 2>&1 || exit 1
for sa in 7 8 9 10; do
  GK_STOP_AFTER=$sa timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfs_persistent -s 0 -c 1 -o gpurun_out/k27_stop$sa python tools/ncu_one.py --config kron27 --runs 1 > gpurun_out/ncu_k27_$sa.log 2>&1
done
for sa in 10 11; do
  GK_STOP_AFTER=$sa timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfs_persistent -s 0 -c 1 -o gpurun_out/u27_stop$sa python tools/ncu_one.py --config urand27 --runs 1 > gpurun_out/ncu_u27_$sa.log 2>&1
done
