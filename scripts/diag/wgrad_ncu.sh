python scripts/wgrad_micro.py
for nm in l4.conv2 l1.conv2; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_ws_kernel -c 1 \
  -o gpurun_out/wgrad_$nm -f python scripts/wgrad_micro.py $nm --ncu > gpurun_out/ncu_wgrad_$nm.log 2>&1; echo "ncu $nm rc=$?"
done
