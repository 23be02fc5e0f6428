#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout ${SWEEP_TIMEOUT:-1500} python scripts/kernel_sweep.py ${SWEEP_ARGS} > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"
tail -12 gpurun_out/sweep.err
