cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/split.jsonl
cp paper_2004_08962_b200/libhicu_b200.so /tmp/lib_g3.so
for g in 2 3 4 5; do
  if [ $g == 3 ]; then cp /tmp/lib_g3.so paper_2004_08962_b200/libhicu_b200.so; else cp varlibs/libhicu_g$g.so paper_2004_08962_b200/libhicu_b200.so; fi
  echo "gps $g" >> gpurun_out/split.jsonl
  timeout 300 python scripts/conv_tc_split2.py >> gpurun_out/split.jsonl 2>>gpurun_out/split.err
done
cp /tmp/lib_g3.so paper_2004_08962_b200/libhicu_b200.so
cat gpurun_out/split.jsonl; tail -3 gpurun_out/split.err
