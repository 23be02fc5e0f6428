cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
python -c "
from paper_2507_22195_b200 import _native as N
for i in range(3): print('fp64 FMA GFLOP/s %.0f   DMMA GFLOP/s %.0f' % (N.fp64_probe(0), N.dmma_probe(0)))
"
