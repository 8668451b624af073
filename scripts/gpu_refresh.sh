#!/bin/bash
# Refresh the committed measurements of the final build: bench lines (bf16, fp8, no-pipeline),
# the config-5 grid at G = 1 (bf16 + fp8), the config-4 shard, the Table-A.5 grid.
mkdir -p gpurun_out
python bench.py > gpurun_out/rf_bench.json 2> gpurun_out/rf_bench.err; echo bench rc=$?
python bench.py --offsets fp8 > gpurun_out/rf_bench_fp8.json 2> gpurun_out/rf_bench_fp8.err; echo bench8 rc=$?
python bench.py --no-pipeline --no-cpu-baseline > gpurun_out/rf_bench_nopipe.json 2>&1; echo benchnp rc=$?
timeout 900 python scripts/sweep.py --grid full > gpurun_out/rf_sweep.jsonl 2> gpurun_out/rf_sweep.err; echo sweep rc=$?
timeout 900 python scripts/sweep.py --grid full --offsets fp8 > gpurun_out/rf_sweep_fp8.jsonl 2> gpurun_out/rf_sweep_fp8.err; echo sweep8 rc=$?
python scripts/config4_bench.py > gpurun_out/rf_config4.json 2> gpurun_out/rf_config4.err; echo c4 rc=$?
ls -la gpurun_out
timeout 600 python scripts/sweep.py --grid paper > gpurun_out/rf_sweep_paper.jsonl 2> gpurun_out/rf_sweep_paper.err; echo sweepp rc=$?
