# round-1 evidence: GPU tests, ncu launch lists + one --set full capture (layer 0's four fused
# launches) per config, ncu traffic -> profiles/ncu_traffic.json, then the bench lines
set -u
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3 > gpurun_out/pytest.txt
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
timeout 600 python bench.py --config q_proj --no-cpu-baseline > gpurun_out/bench_q_proj.json 2> gpurun_out/bench_q_proj.err
