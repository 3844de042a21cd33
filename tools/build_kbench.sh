# Builds the k_train micro-benchmark variants (development tool; run on the GPU box or here).
#   bash tools/build_kbench.sh <name> [extra nvcc flags...]   -> tools/kbench_<name>
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo ${KB_PT--DNFG_PHASE_TIMING} "$@" \
    -I paper_2201_05989_b200/csrc tools/kbench.cu paper_2201_05989_b200/csrc/aux_kernels.cu \
    paper_2201_05989_b200/csrc/host_init.cpp -o tools/kbench_$NAME
