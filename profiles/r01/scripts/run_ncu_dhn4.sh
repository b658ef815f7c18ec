mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dhn4_kernel -s 1 -c 1 -o /tmp/ncu/dhn4 -f python profiles/probe_dhn.py 0.1 > gpurun_out/ncu_dhn4.log 2>&1
ncu -i /tmp/ncu/dhn4.ncu-rep --page raw --csv > gpurun_out/prof_dhn4_raw.csv 2>&1
ncu -i /tmp/ncu/dhn4.ncu-rep --page source --csv > gpurun_out/prof_dhn4_source.csv 2>&1
ncu -i /tmp/ncu/dhn4.ncu-rep --page details --csv > gpurun_out/prof_dhn4_details.csv 2>&1
