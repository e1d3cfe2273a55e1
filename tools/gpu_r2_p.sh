set -x
timeout 900 python tools/setup_time.py 16777216 3 gaussian recompute 2 > gpurun_out/setup_c4_r2p.log 2>&1; cat gpurun_out/setup_c4_r2p.log | tail -2
timeout 600 python tools/setup_time.py 4194304 4 gaussian recompute 2 > gpurun_out/setup_c5_r2p.log 2>&1; tail -1 gpurun_out/setup_c5_r2p.log
timeout 900 python tools/c5_cg.py 262144 4 300 exact > gpurun_out/c5cg_2e18_r2p.log 2>&1; tail -1 gpurun_out/c5cg_2e18_r2p.log | cut -c 1-700
timeout 900 python tools/c5_cg.py 1048576 4 300 exact > gpurun_out/c5cg_2e20_r2p.log 2>&1; tail -1 gpurun_out/c5cg_2e20_r2p.log | cut -c 1-700
