#!/usr/bin/env bash
# round 2: default bench line (config 3) + reference arm + partitioned N=1 A/B
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python bench.py --partitioned --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_part1.json 2> gpurun_out/bench_part1.err; echo "part rc=$?"
tail -c 600 gpurun_out/bench.json; tail -c 300 gpurun_out/bench_ref.json; tail -c 600 gpurun_out/bench_part1.json
