# final 1-GPU evidence for the round (each step logged separately)
python -m pytest tests -m gpu -q --timeout 1500 --ignore=tests/test_gpu_multi.py -rf > gpurun_out/final_gputest.log 2>&1; echo rc=$? >> gpurun_out/final_gputest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo rc=$? >> gpurun_out/final_bench_n1.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python bench.py --only-headline --no-e2e --no-cpu --steps 3 --sweep-n > gpurun_out/final_smalln_n1.json 2> gpurun_out/final_smalln_n1.err
bash tools/profile.sh r02final > gpurun_out/prof_r02final_steps.txt 2>&1
