# Context / budget sweep of the headline decode step (B = 1, 32 layers,
# 32Q/8KV): one bench line per point, summarised by tools/sweep_summary.py.
mkdir -p gpurun_out/sweep
for S in 32768 65536 131072; do
  for BU in 1024 2048 4096 8192; do
    timeout 300 python bench.py --seq $S --budget $BU --steps 10 --warmup 3 --no-extra --no-prefill \
      --no-cpu-baseline > gpurun_out/sweep/s${S}_b${BU}.json 2>/dev/null
  done
done
python tools/sweep_summary.py gpurun_out/sweep
