L=paper_2307_07950_b200/_lib
cp $L/libselsync_b200.so /tmp/varF.so
for V in F B F B; do
  if [ $V = F ]; then cp /tmp/varF.so $L/libselsync_b200.so; else cp $L/var$V/libselsync_b200.so $L/libselsync_b200.so; fi
  echo "== var$V"
  timeout 300 python tools/step_kernel_solo.py update_first local 2>&1 | grep "order="
  GRAPH=1 timeout 300 python tools/step_kernel_solo.py update_first local 1000000 2>&1 | grep "order="
done
cp /tmp/varF.so $L/libselsync_b200.so
timeout 300 python tools/step_kernel_solo.py update_first sync 2>&1 | grep "order="
