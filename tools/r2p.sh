mkdir -p gpurun_out
VXG_FOLD_MERGED=0 VXG_FOLD_SERIAL=1 timeout 200 python tools/probe_fold.py > gpurun_out/r2p_probe_serial.txt 2>&1
VXG_FOLD_MERGED=0 timeout 200 python tools/probe_fold.py > gpurun_out/r2p_probe_unmerged.txt 2>&1
