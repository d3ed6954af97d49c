set -x
for ch in 100 50 34 25 20 14 10; do
  echo "== chunk $ch" >> gpurun_out/r02aj_chunk.txt
  GX_SAMPLER_CHUNK=$ch GX_SAMPLER_TRACE=1 timeout 300 python bench.py --steps 6 --warmup 4 --no-cpu-baseline --no-tiers --pressure-frac 0 > gpurun_out/r02aj_chunk_$ch.json 2> gpurun_out/r02aj_chunk_$ch.err
  python - <<PY >> gpurun_out/r02aj_chunk.txt
import json
d=json.loads(open("gpurun_out/r02aj_chunk_$ch.json").read().strip().splitlines()[-1])
print($ch, d["ms_per_step"], d["stages"]["sample_ms"])
PY
  grep "sampler trace" gpurun_out/r02aj_chunk_$ch.err | tail -n 3 >> gpurun_out/r02aj_chunk.txt
done
