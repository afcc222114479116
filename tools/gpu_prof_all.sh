# ncu --set full of every launch of one warm C2 raster step (prof_workload runs a warm-up
# step first; -s skips its launches), plus the launch-time list
python tools/prof_workload.py raster c2 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_raster.csv python tools/prof_workload.py raster c2 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_raster|k_bwd|k_emit|k_ranges|k_splat' -s 14 -c 20 -f -o gpurun_out/raster_all python tools/prof_workload.py raster c2 1 > gpurun_out/ncu_raster_all.log 2>&1
tail -2 gpurun_out/ncu_raster_all.log
