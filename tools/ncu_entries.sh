# ncu --set full captures of selected plan entries (gpurun), third launch of each (L2 warm from the
# previous two). Usage: bash tools/ncu_entries.sh TAG PLAN "4:dwpw_tc 16:dwpw_tc 13:pw_tc"
TAG=$1; PLAN=$2; shift 2
for ek in $1; do
  e=${ek%%:*}; k=${ek##*:}
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/${TAG}_e$e \
    python tools/prof_entry.py --entries $e --reps 3 --plan-file $PLAN > gpurun_out/${TAG}_e$e.log 2>&1
done
ls gpurun_out
