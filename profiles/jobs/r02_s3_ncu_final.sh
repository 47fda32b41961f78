# round 2, session 3: ncu launch list + --set full of the decode fused launches on the final (12-warp) build
set -u
O=gpurun_out/s3ncuf
mkdir -p $O
bash profiles/run_ncu.sh s3f5 decode > /dev/null 2>&1
mv gpurun_out/s3f5_decode_launches.csv gpurun_out/s3f5_decode_apply_fused_kernel.ncu-rep $O/ 2>/dev/null
python profiles/summarize_ncu.py $O/s3f5_decode_apply_fused_kernel.ncu-rep > $O/s3f5_decode_fused_summary.txt 2>&1; cat $O/s3f5_decode_fused_summary.txt
ncu -i $O/s3f5_decode_apply_fused_kernel.ncu-rep --page raw --csv > $O/s3f5_decode_fused_raw.csv 2>/dev/null; wc -l $O/s3f5_decode_fused_raw.csv
