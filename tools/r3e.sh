mkdir -p gpurun_out
timeout 200 python tools/probe_f1.py 0 4 > gpurun_out/r3e_f1_cfg0.txt 2>&1
timeout 200 python tools/probe_f1.py 1 4 > gpurun_out/r3e_f1_cfg1.txt 2>&1
bash tools/ab_libs.sh default tools/libvxg_ring6.so tools/libvxg_long3072.so tools/libvxg_long5120.so default > gpurun_out/r3e_ab.log 2>&1
