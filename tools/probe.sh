set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | head -20; free -g
(nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &) ; 
./tools/fp64_peak | tee gpurun_out/fp64_peak.json
sleep 0.5
./tools/fp64_peak | tee -a gpurun_out/fp64_peak.json
