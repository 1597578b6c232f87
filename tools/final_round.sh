set -x
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/final/smoke.log
python -m pytest tests -m gpu -q -x -rA > gpurun_out/final/gpu_tests.log 2>&1; tail -3 gpurun_out/final/gpu_tests.log
python bench.py > gpurun_out/final/bench_k27.json 2> gpurun_out/final/bench_k27.err
python bench.py --impl reference --steps 8 --warmup 3 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
python bench.py --config urand27 --steps 16 > gpurun_out/final/bench_u27.json 2> gpurun_out/final/bench_u27.err
python bench.py --config kron16 --steps 64 > gpurun_out/final/bench_k16.json 2> gpurun_out/final/bench_k16.err
python bench.py --config grid4900 --steps 8 > gpurun_out/final/bench_grid.json 2> gpurun_out/final/bench_grid.err
