# Quick GPU check (gpurun): parity subset + default bench. Usage: bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}; K=${2:-"dwpw or pwdw or steady or network"}
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" 2>&1 | tail -15 > gpurun_out/${TAG}_gputest.txt
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-cudnn --no-energy --plan-out gpurun_out/${TAG}_plan.json > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_gputest.txt; python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench.json'));print(d['value'],d['ms_per_step'],d['roofline'])"
