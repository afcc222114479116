# usage: bash tools/gpu_prof.sh <kernel-regex> <tag> [workload] [cfg]
ncu --set full --clock-control none --import-source on -k regex:$1 -s 1 -c 1 -f -o gpurun_out/$2 python tools/prof_workload.py ${3:-raster} ${4:-c2} 1 > gpurun_out/ncu_$2.log 2>&1
tail -1 gpurun_out/ncu_$2.log
