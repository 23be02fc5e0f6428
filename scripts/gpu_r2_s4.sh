#!/usr/bin/env bash
timeout 900 python -m pytest tests/test_gpu_integration.py tests/test_gpu_pdl.py -q 2>&1 | tail -15
# ncu --set full of the config-3 operator step kernels (traffic for the roofline line)
python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-implicit --no-cpu-baseline > gpurun_out/b3s.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_face2|k_local_solve|k_precond_apply|k_residual" -s 4 -c 8 \
    -o gpurun_out/prof_cfg3 python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-implicit --no-cpu-baseline > gpurun_out/ncu_full3.log 2>&1
echo "ncu rc=$?"
