# ncu --set full of bfs_persistent stopped after barriers $STOPS (GK_STOP_AFTER), first kron27 bench source
for sa in $STOPS; do
  GK_STOP_AFTER=$sa timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfs_persistent -s 0 -c 1 -o gpurun_out/${TAG}_stop$sa python tools/ncu_one.py --config ${CFG:-kron27} --runs 1 > gpurun_out/ncu_${TAG}_$sa.log 2>&1
done
