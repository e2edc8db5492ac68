timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for f in 0 1; do RNNTG_FUSED_PE=$f timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench27_$f.json 2> gpurun_out/bench27_$f.err; python -c "
import json;d=json.load(open('gpurun_out/bench27_$f.json'));print($f, {k:d.get(k) for k in ['value','ms_per_step','decode_kernel_ms','e2e']})"; done
