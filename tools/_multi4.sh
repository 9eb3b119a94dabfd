# 4-GPU evidence: the multi-GPU tests, the driver-style bench line (exchange latency at
# 8 B..16 KB), and the small-n sweep (the paper's latency regime) under torchrun
python -m pytest tests/test_gpu_multi.py -v --timeout 1500 > gpurun_out/r02_multi4.log 2>&1; echo rc=$? >> gpurun_out/r02_multi4.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 5 --no-sweep > gpurun_out/r02_bench_n4.json 2> gpurun_out/r02_bench_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 3 --only-headline --no-e2e --sweep-n > gpurun_out/r02_smalln_n4.json 2> gpurun_out/r02_smalln_n4.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 --no-sweep > gpurun_out/r02_bench_n2.json 2> gpurun_out/r02_bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --steps 3 --only-headline --no-e2e --sweep-n > gpurun_out/r02_smalln_n2.json 2> gpurun_out/r02_smalln_n2.err
