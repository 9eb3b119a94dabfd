# small-n A/B, round-1 build vs current (bench --sweep-n: CUDA events around aa_step only)
for lib in build/libaa_r1.so paper_2110_09667_b200/libaa.so; do
  AA_LIB=$lib timeout 600 python bench.py --only-headline --no-e2e --no-cpu --steps 3 --sweep-n > gpurun_out/smalln_$(basename $lib .so).json 2>gpurun_out/smalln_$(basename $lib .so).err
done
python tools/graph_probe.py 1000,100000 20 > gpurun_out/r02_graph_probe.txt 2>&1
python -m pytest tests/test_gpu_graph.py -q -x > gpurun_out/r02_graph_test.log 2>&1; echo rc=$? >> gpurun_out/r02_graph_test.log
python tools/timeline_probe.py 1000 20 dcgs2 > gpurun_out/r02_timeline7.txt 2>&1
