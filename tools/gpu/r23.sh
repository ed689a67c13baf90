mkdir -p gpurun_out/r23
cp paper_2511_00737_b200/libephdc.so /tmp/lib_orig.so
cp ablibs/libDBG.so paper_2511_00737_b200/libephdc.so
for rep in 1 2 3 4; do
  echo "== rep $rep"
  timeout 120 python tools/c5_point.py --lg 16 --L 9 --bits 30 --op inv --batch 7281 --reps 100 2>&1 | grep -E "c5 wait|GB_s|Error" | sort | uniq -c | head -20
done
for rep in 1 2; do
  echo "== 14 rep $rep"
  timeout 120 python tools/c5_point.py --lg 14 --L 3 --bits 48 --op inv --batch 65536 --reps 100 2>&1 | grep -E "c5 wait|GB_s|Error" | sort | uniq -c | head -20
done
cp /tmp/lib_orig.so paper_2511_00737_b200/libephdc.so
