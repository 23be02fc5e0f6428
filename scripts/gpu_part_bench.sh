#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python bench.py --partitioned --steps 50 --warmup 3 --e2e-steps 5 > gpurun_out/pb1.json 2> gpurun_out/pb1.err; echo "part N=1 rc=$?"; cut -c1-600 gpurun_out/pb1.json; tail -3 gpurun_out/pb1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --backend gloo --ncells 8 --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/pb2.json 2> gpurun_out/pb2.err; echo "part gloo N=2 rc=$?"; cut -c1-600 gpurun_out/pb2.json; tail -5 gpurun_out/pb2.err
