#!/bin/bash
# Configuration sweep on one B200 with per-kernel-class timing (bench.py lines into $1/):
# the `kernels` field gives each class's in-step TF/s or GB/s (timed in a serialised extra run).
#   bash scripts/sweep_kt.sh gpurun_out/sweep_kt
out=${1:-gpurun_out/sweep_kt}
mkdir -p "$out"
run() { name=$1; shift; timeout 900 python bench.py "$@" > "$out/$name.json" 2> "$out/$name.err"; }
run 1p3b_d8 --model 1p3b --depth 8 --threshold 32
run 350m_d2 --model 350m --depth 2 --threshold 16
run 350m_d4 --model 350m --depth 4 --threshold 16
run bert_d8 --model bert --depth 8 --threshold 32
run 2p7b_d2 --model 2p7b --depth 2 --threshold 8
run 2p7b_d4 --model 2p7b --depth 4 --threshold 16
run 2p7b_d8 --model 2p7b --depth 8 --threshold 32 --recompute
python bench.py --impl reference > "$out/reference_arm.json" 2> "$out/reference_arm.err"
