mkdir -p gpurun_out
./tools/micro/burst > gpurun_out/burst_main.txt 2>&1
BURST2=1 ./tools/micro/burst > gpurun_out/burst2.txt 2>&1
BURST3=1 ./tools/micro/burst > gpurun_out/burst3.txt 2>&1
SKB_DEBUG_TIMING=1 python paper_2605_08575_b200/build.py --force 2>&1 | grep -i error
timeout 120 python tools/dbg_dec.py olmoe 1 > gpurun_out/dbg_olmoe1.txt 2>&1
tail -40 gpurun_out/dbg_olmoe1.txt
