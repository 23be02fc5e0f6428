#!/usr/bin/env bash
timeout 900 python bench.py --m 2 --ncells 16 --steps 10 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/bench_m2.json 2> gpurun_out/bench_m2.err; echo "rc=$?"
tail -c 1500 gpurun_out/bench_m2.json; tail -5 gpurun_out/bench_m2.err
