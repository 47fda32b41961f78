# compute-sanitizer over every apply path plus the round-2 additions (JD-Diag, page-in, tensor-core JD)
set -u
O=gpurun_out/s2x
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool python profiles/microbench/sanitize_apply.py > $O/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> $O/sanitize_$tool.txt
  tail -3 $O/sanitize_$tool.txt
done
grep -h "Race reported\|Error:" $O/sanitize_racecheck.txt | sort | uniq -c | head
