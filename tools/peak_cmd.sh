nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 250 > gpurun_out/peak_clocks.csv &
SMI=$!
python tools/fp64_peak.py > gpurun_out/fp64_peak.json 2> gpurun_out/fp64_peak.err
kill $SMI
nvidia-smi -q | head -60 > gpurun_out/nvsmi.txt
cat gpurun_out/fp64_peak.json
