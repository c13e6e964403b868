# Build + run the DW-core variant microbenchmark on a B200 (gpurun): bash tools/microbench/run_variants.sh
set -e
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2404_19331_b200/csrc -I ../../include --expt-relaxed-constexpr -o /tmp/dwv dw_core_variants.cu
/tmp/dwv | tee ../../gpurun_out/dw_core_variants.txt
[ -n "$SKIP_FFO" ] && exit 0
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ffo ffma2_operands.cu
/tmp/ffo | tee ../../gpurun_out/ffma2_operands.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/opc op_costs.cu
/tmp/opc | tee ../../gpurun_out/op_costs.txt
