# Round-2 first evidence run on a B200 (gpurun): GPU tests, smoke, default bench with plan / per-layer output.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r02a_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.txt 2>&1
timeout 900 python bench.py --plan-out gpurun_out/r02a_plan.json --layers-out gpurun_out/r02a_layers.json > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
ls gpurun_out
