# local-t decode path: GPU suite, bench lines, A/B against CTS_LOCAL_T=0, per-CTA timeline
set -u
O=gpurun_out/s2i
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
tail -3 $O/pytest.txt
for c in decode multi prefill diag_decode; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -shared -ldl"
cp paper_2407_00066_b200/libcts.so /tmp/keep.so
$NV -DCTS_LOCAL_T=0 -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python bench.py --config decode --no-cpu-baseline > $O/bench_decode_old.json 2>> $O/bench.err
timeout 300 python bench.py --config multi --no-cpu-baseline > $O/bench_multi_old.json 2>> $O/bench.err
$NV -DCTS_TRACE -o paper_2407_00066_b200/libcts.so paper_2407_00066_b200/csrc/cts.cu
timeout 300 python profiles/microbench/trace_fused.py > $O/trace_localt.txt 2>&1
cp /tmp/keep.so paper_2407_00066_b200/libcts.so
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['roofline']['frac'] if 'roofline' in d else '', d.get('clocks',{}).get('sm_mhz'))"; done
