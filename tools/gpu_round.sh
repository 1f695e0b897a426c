#!/bin/bash
# One GPU session: tests, smoke, bench (+ reference arm), per-config timings
# with clocks, ncu launch list.  Usage: tools/gpu_round.sh TAG
T=${1:-r02x}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_tests.log 2>&1; tail -3 $O/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; tail -2 $O/${T}_smoke.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; tail -c 300 $O/${T}_bench.json
timeout 600 python bench.py --impl reference > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err; tail -c 200 $O/${T}_bench_ref.json
timeout 900 python tools/bench_configs.py > $O/${T}_configs.jsonl 2> $O/${T}_configs.err; wc -l $O/${T}_configs.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/${T}_ncu.log 2>&1; wc -l $O/${T}_launches.csv
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${T}_smi.txt 2>&1
