# Round-end evidence run (on a B200 via gpurun): GPU tests, default bench, smoke, per-config bench lines, ncu captures.
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --plan-out gpurun_out/plan_measured.json --layers-out gpurun_out/r01_layers.json > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01_smoke.txt 2>&1
for cfg in "mobilenet_v1 s8 64" "efficientnet_b0 s8 256" "cvt13 bf16 512" "mobilenet_v2 bf16 1" "single_dwpw f32 1" "single_dwpw s8 1" "xception bf16 64" "xception s8 64" "proxylessnas_gpu bf16 64" "proxylessnas_gpu s8 64" "ceit_leff bf16 256" "cmt_irffn bf16 128" "cmt_irffn s8 128"; do
  set -- $cfg
  timeout 400 python bench.py --net $1 --dtype $2 --batch $3 --steps 50 --warmup 5 --no-cpu-baseline --plan-out gpurun_out/plan_$1_$2_$3.json > gpurun_out/bench_$1_$2_$3.json 2>gpurun_out/bench_$1_$2_$3.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_raw.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-cudnn --no-energy > /dev/null 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control all --clock-control none --csv --log-file gpurun_out/r01_dram.csv python tools/prof_entry.py --entries all --reps 1 --plan-file gpurun_out/plan_measured.json > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:dwpw -s 2 -c 1 -o gpurun_out/r01_dwpw python tools/prof_entry.py --entries 4 --reps 3 --plan-file gpurun_out/plan_measured.json > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:dw_nhwc -s 3 -c 1 -o gpurun_out/r01_dw_i8 python tools/prof_dw.py 64 56 128 8 16 > /dev/null 2>&1
ls gpurun_out
