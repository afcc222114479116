# round-end evidence: GPU tests, smoke, bench line, ncu captures (raster + voxel steps)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_raster.csv python tools/prof_workload.py raster c2 1 > /dev/null 2>&1
RS=$(python tools/ncu_skip.py gpurun_out/launches_raster.csv 'k_raster|k_bwd|k_emit|k_ranges|k_splat')
ncu --set full --clock-control none --import-source on -k regex:'k_raster|k_bwd|k_emit|k_ranges|k_splat' $RS -f -o gpurun_out/raster_all python tools/prof_workload.py raster c2 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_voxel.csv python tools/prof_workload.py voxel c3 1 > /dev/null 2>&1
VS=$(python tools/ncu_skip.py gpurun_out/launches_voxel.csv 'k_voxel|k_emit_brick')
ncu --set full --clock-control none --import-source on -k regex:'k_voxel|k_emit_brick' $VS -f -o gpurun_out/voxel_all python tools/prof_workload.py voxel c3 1 > /dev/null 2>&1
ls -la gpurun_out
