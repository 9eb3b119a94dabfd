set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_breakdown.py tests/test_gpu_step_host.py -q -x > gpurun_out/r02_tma_tests.log 2>&1; echo rc=$? >> gpurun_out/r02_tma_tests.log
for r in 1 2; do
AA_K1_STORE=0 timeout 600 python bench.py --steps 10 --no-e2e --no-cpu --sweep > gpurun_out/r02_ab_stg_$r.json 2>gpurun_out/r02_ab_stg_$r.err
AA_K1_STORE=1 timeout 600 python bench.py --steps 10 --no-e2e --no-cpu --sweep > gpurun_out/r02_ab_tma_$r.json 2>gpurun_out/r02_ab_tma_$r.err
done
