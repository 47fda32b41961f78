set -u
O=gpurun_out/s2z2
mkdir -p $O
for rep in 1; do
for v in old new; do
  cp ab/libcts_$v.so paper_2407_00066_b200/libcts.so
  for it in 10 50; do echo -n "$v rep$rep: " >> $O/ab.txt; timeout 300 python profiles/microbench/jd_speed.py $it 2>&1 | tail -1 >> $O/ab.txt; done
done
done
cat $O/ab.txt
