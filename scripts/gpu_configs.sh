#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python scripts/implicit_step.py --case tgv --n 16 --p 3 --flux kepes --dt 0.57 --viscous > gpurun_out/cfg4_n16.json 2> gpurun_out/cfg4_n16.err
python -c "
import json; d=json.load(open('gpurun_out/cfg4_n16.json')); print({k:v for k,v in d.items() if k!='records'})" || tail -3 gpurun_out/cfg4_n16.err
timeout 900 python scripts/implicit_step.py --case tgv --n 32 --p 3 --flux kepes --dt 0.057 > gpurun_out/cfg3_dt0057.json 2> gpurun_out/cfg3_dt0057.err
python -c "
import json; d=json.load(open('gpurun_out/cfg3_dt0057.json')); print({k:v for k,v in d.items() if k!='records'})" || tail -3 gpurun_out/cfg3_dt0057.err
