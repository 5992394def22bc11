nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 1000 > gpurun_out/sustain_clocks.csv &
SMI=$!
for i in 1 2 3 4 5 6; do timeout 300 python scripts/spmm_time.py 16384; done
kill $SMI
cat gpurun_out/sustain_clocks.csv | awk 'NR%4==1'
