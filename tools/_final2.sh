# 2-GPU box: the driver-style default bench under torchrun (sweep included), then the whole GPU suite
start=$(date +%s)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02_bench_n2_default.json 2> gpurun_out/r02_bench_n2_default.err; echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r02_bench_n2_default.err
python -m pytest tests -m gpu -q --timeout 1500 -rf > gpurun_out/r02_gputest_all2.log 2>&1; echo rc=$? >> gpurun_out/r02_gputest_all2.log
