#!/bin/bash
# ncu --set full on one kernel regex ($KREGEX) of the short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
SHORT="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 2"
$SHORT > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${KSKIP:-0} -c ${KCOUNT:-1} -o gpurun_out/${KOUT:-prof} $SHORT > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_full.log
