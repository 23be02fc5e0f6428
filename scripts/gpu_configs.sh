#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python scripts/krylov_profile.py --viscous 2>&1 | tail -3
timeout 300 python scripts/krylov_profile.py 2>&1 | tail -3
timeout 900 python scripts/implicit_step.py --case tgv --n 32 --p 3 --flux kepes --dt 0.57 > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err
tail -5 gpurun_out/cfg3.err
python -c "
import json; d=json.load(open('gpurun_out/cfg3.json')); print({k:v for k,v in d.items() if k!='records'})"
