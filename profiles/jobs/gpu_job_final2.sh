# round-1 evidence sweep (third pass, after the 256-bit accesses): tests, smoke, ncu, bench lines
set -u
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
rm -f profiles/ncu_traffic.json
for c in decode prefill; do
  timeout 900 bash profiles/run_ncu.sh r01 $c > gpurun_out/ncu_$c.log 2>&1
  W=$(python -c "import bench; print(bench.CONFIGS['$c']['workload'])")
  python profiles/make_traffic.py $W gpurun_out/r01_${c}_apply_fused_kernel.ncu-rep gpurun_out/${W}_alg_bytes.json >> gpurun_out/ncu_$c.log 2>&1
  python profiles/summarize_ncu.py gpurun_out/r01_${c}_apply_fused_kernel.ncu-rep > gpurun_out/r01_${c}_fused_summary.txt 2>&1
done
cp profiles/ncu_traffic.json gpurun_out/ 2>/dev/null
timeout 600 python bench.py > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err
timeout 600 python bench.py --config prefill --no-cpu-baseline > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err
timeout 600 python bench.py --config multi --no-cpu-baseline > gpurun_out/bench_multi.json 2> gpurun_out/bench_multi.err
timeout 900 python bench.py --config proj_prefill > gpurun_out/bench_proj_prefill.json 2> gpurun_out/bench_proj_prefill.err
timeout 900 python bench.py --config lora_decode --no-cpu-baseline > gpurun_out/bench_lora_decode.json 2> gpurun_out/bench_lora_decode.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 python profiles/microbench/jd_speed.py 10 > gpurun_out/jd_speed.txt 2>&1
