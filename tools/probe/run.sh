nproc; free -g; lscpu | grep -E "Model name|Socket|Thread|Core"; nvidia-smi; 
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probe/fp64_peak | tee gpurun_out/probe.log
kill $SMI
