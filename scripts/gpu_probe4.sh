timeout 120 build/nvlink_probe 512 > gpurun_out/nvlink_probe_g4.log 2>&1; echo probe=$?; cat gpurun_out/nvlink_probe_g4.log
