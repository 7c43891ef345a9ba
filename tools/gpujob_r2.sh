# Round-2 final GPU job: smoke, the GPU suite, the bench line, the headline's
# launch list and one full ncu capture of the fused layer (run under gpurun).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_decode_fused|k_score_blocks|k_select_reg|k_decode_attn" -c 200 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --no-extra --no-prefill --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
