#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_entropy.py -q 2>&1 | tail -15
timeout 1500 python scripts/h_sweep.py --n 8 --levels 3 > gpurun_out/hsweep.json 2> gpurun_out/hsweep.err; echo "hsweep rc=$?"
tail -4 gpurun_out/hsweep.json
