# End-of-round measurement set: full (tests, smoke, bench, reference arm, ncu), configs, f16, batch sweep, stage units.
set -x
tag=${1:-final}
bash tools/gpu_full.sh ${tag}
timeout 600 python bench.py --no-cpu --dtype f16 > gpurun_out/${tag}_f16.json 2> gpurun_out/${tag}_f16.err; echo f16=$?
bash tools/gpu_configs.sh
for c in cfg2 cfg3 cfg4; do cp gpurun_out/$c.json gpurun_out/${tag}_$c.json; done
for b in 1 4 8 16 32; do
  timeout 300 python bench.py --no-cpu --batch $b --steps 20 > gpurun_out/${tag}_sweep_b$b.json 2> gpurun_out/${tag}_sweep_b$b.err; echo sweep$b=$?
done
timeout 600 python tools/bench_units.py > gpurun_out/${tag}_units.jsonl 2> gpurun_out/${tag}_units.err; echo units=$?
