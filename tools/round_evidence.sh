# Round-end evidence run (on a B200 via gpurun): GPU tests, smoke, default bench, per-config bench lines,
# ncu launch list, per-entry DRAM traffic of the executed plan and of the all-LBL plan (FCM savings),
# ncu --set full captures. Usage: bash tools/round_evidence.sh [TAG]
T=${1:-r02}
O=gpurun_out/$T
mkdir -p $O/configs
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > $O/gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py --plan-out $O/plan_measured.json --layers-out $O/layers.json > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for cfg in "mobilenet_v2 f32 64" "mobilenet_v1 s8 64" "mobilenet_v1 bf16 64" "efficientnet_b0 s8 256" "cvt13 bf16 512" "mobilenet_v2 bf16 1" "mobilenet_v2 bf16 64" "single_dwpw f32 1" "single_dwpw s8 1" "xception bf16 64" "xception s8 64" "proxylessnas_gpu bf16 64" "proxylessnas_gpu s8 64" "ceit_leff bf16 256" "cmt_irffn bf16 128" "cmt_irffn s8 128" "efficientnet_b0 bf16 256"; do
  set -- $cfg
  timeout 400 python bench.py --net $1 --dtype $2 --batch $3 --steps 50 --warmup 5 --no-cpu-baseline --plan-out $O/configs/plan_$1_$2_$3.json > $O/configs/bench_$1_$2_$3.json 2> $O/configs/bench_$1_$2_$3.err
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench_raw.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-cudnn --no-energy > /dev/null 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,gpu__time_duration.sum
timeout 400 ncu --metrics $M --cache-control all --clock-control none --csv --log-file $O/entries_fused.csv python tools/prof_entry.py --entries all --reps 1 --plan-file $O/plan_measured.json > /dev/null 2>&1
timeout 400 ncu --metrics $M --cache-control all --clock-control none --csv --log-file $O/entries_lbl.csv python tools/prof_entry.py --entries all --reps 1 --plan-file $O/plan_measured.json --lbl --plan-out $O/plan_lbl.json > /dev/null 2>&1
python tools/ncu_savings.py $O/entries_fused.csv $O/plan_measured.json $O/entries_lbl.csv $O/plan_lbl.json $O/ncu_savings.json > $O/ncu_savings.txt 2>&1
E=$(python -c "import json;p=json.load(open('$O/plan_measured.json'));print([i for i,e in enumerate(p['entries']) if e['layers']==['b2.1','b2.2']][0])")
timeout 300 ncu --set full --import-source on --clock-control none -k regex:dwpw -s 1 -c 1 -o $O/ncu_dwpw_b2 python tools/prof_entry.py --entries $E --reps 2 --plan-file $O/plan_measured.json > /dev/null 2>&1
E=$(python -c "import json;p=json.load(open('$O/plan_measured.json'));print([i for i,e in enumerate(p['entries']) if e['op']=='pwdw_r'][0])")
timeout 300 ncu --set full --import-source on --clock-control none -k regex:pwdw -s 1 -c 1 -o $O/ncu_pwdw_b1 python tools/prof_entry.py --entries $E --reps 2 --plan-file $O/plan_measured.json > /dev/null 2>&1
ls -R $O | head -80
