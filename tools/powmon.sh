nvidia-smi -q -d POWER | grep -iE "limit|draw" | head -12
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown --format=csv -lms 20 > gpurun_out/pow.csv &
PID=$!
sleep 0.5
python tools/sweep.py --levels 011102 --reps 200 --tunes "" > gpurun_out/pw_sweep.log 2>&1
kill $PID
