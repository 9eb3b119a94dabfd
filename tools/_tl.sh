python tools/timeline_probe.py 1000 20 dcgs2 > gpurun_out/r02_timeline8.txt 2>&1
python tools/timeline_probe.py 100000 20 dcgs2 >> gpurun_out/r02_timeline8.txt 2>&1
