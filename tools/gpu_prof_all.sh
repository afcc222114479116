set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_raster.csv python tools/prof_workload.py raster c2 1 > /dev/null 2>&1
RS=$(python tools/ncu_skip.py gpurun_out/launches_raster.csv 'k_raster|k_bwd|k_emit|k_ranges|k_splat')
ncu --set full --clock-control none --import-source on -k regex:'k_raster|k_bwd|k_emit|k_ranges|k_splat' $RS -f -o gpurun_out/raster_all python tools/prof_workload.py raster c2 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_voxel.csv python tools/prof_workload.py voxel c3 1 > /dev/null 2>&1
VS=$(python tools/ncu_skip.py gpurun_out/launches_voxel.csv 'k_voxel|k_emit_brick')
ncu --set full --clock-control none --import-source on -k regex:'k_voxel|k_emit_brick' $VS -f -o gpurun_out/voxel_all python tools/prof_workload.py voxel c3 1 > /dev/null 2>&1
ls -la gpurun_out
