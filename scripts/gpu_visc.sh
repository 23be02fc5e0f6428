#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -x -q -k "visc or Visc or steps" 2>&1 | tail -15
timeout 300 python scripts/krylov_profile.py --viscous 2>&1 | tail -2
