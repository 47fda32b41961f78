# round-2 session-3 closing evidence on the final build: GPU suite, smoke, every bench config, reference
# arm, ncu launch list + --set full of the decode fused launches, and of the K-space Gram GEMM
set -u
O=gpurun_out/s3final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 600 python bench.py > $O/bench_decode.json 2>> $O/bench.err
for c in prefill multi q_proj diag_decode lora_decode lora_matched tp_decode proj_prefill; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>> $O/bench.err
for f in $O/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); sys.exit()
r = d.get("roofline", {})
print(f.split("/")[-1], round(d["value"], 1), d["unit"], "frac", r.get("frac"), "ms/step", d.get("ms_per_step"),
      "mhz", d.get("clocks", {}).get("sm_mhz"), "parity", (d.get("parity_check") or {}).get("max_row_rel_err"))
PY
done
for it in 10 50; do timeout 300 python profiles/microbench/jd_speed.py $it >> $O/jd_speed.txt 2>&1; done
cat $O/jd_speed.txt
bash profiles/run_ncu.sh s3 decode > /dev/null 2>&1
mv gpurun_out/s3_decode_launches.csv gpurun_out/s3_decode_apply_fused_kernel.ncu-rep $O/ 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"jd_tc_gemm<128>|jd_tc_gemmILi128" -c 1 -o $O/s3_jd_gram_gemm python profiles/microbench/jd_speed.py 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:jd_ --csv --log-file $O/s3_jd_launches.csv python profiles/microbench/jd_speed.py 10 > /dev/null 2>&1
python profiles/summarize_ncu.py $O/s3_decode_apply_fused_kernel.ncu-rep > $O/s3_decode_fused_summary.txt 2>&1
python profiles/summarize_ncu.py $O/s3_jd_gram_gemm.ncu-rep > $O/s3_jd_gram_summary.txt 2>&1
cat $O/s3_decode_fused_summary.txt $O/s3_jd_gram_summary.txt | head -20
ls -la $O
