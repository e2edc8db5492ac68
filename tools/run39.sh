# Time-sliced host-frame path: parity tests, then the bench's e2e with the
# sliced path (default), the fused path, and slice-length variants.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sliced.py tests/test_gpu_fused.py -q -x --timeout 300 2>&1 | tail -3
for v in "" "RNNTG_SLICED=0" "RNNTG_SLICE_FIRST=32 RNNTG_SLICE_MAX=128" "RNNTG_SLICE_FIRST=8 RNNTG_SLICE_MAX=512"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b39.json 2> gpurun_out/b39.err
  echo "[$v]"; python -c "
import json;d=json.load(open('gpurun_out/b39.json'));print(round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), d['decode_kernel_ms'], d['ms_per_step'])"
done
