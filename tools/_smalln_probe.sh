# small-n latency evidence (1 GPU): host enqueue cost, phase timeline, step latency
python tools/host_overhead.py > gpurun_out/r02_host_overhead.txt 2>&1
python tools/timeline_probe.py 1000 20 dcgs2 > gpurun_out/r02_timeline.txt 2>&1
python tools/step_latency.py 1000,100000 20 > gpurun_out/r02_step_latency.txt 2>&1
