#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
CMD="python scripts/implicit_step.py --n 16 --p 3"
$CMD > gpurun_out/step_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv $CMD > gpurun_out/ncu_step.log 2>&1; echo "ncu rc=$?"
