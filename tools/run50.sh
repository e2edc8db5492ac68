for b in 128 256 512; do
RNNTG_SLICED=1 timeout 300 python tools/prof_beam.py $b 500 3 | python -c "import json,sys;d=json.load(sys.stdin);print('B=$b', d['decode_ms'], d['gpu_ms'], 'rows/sf', round(d['rows_per_sf'],2), 'phase', d['phase_share'], 'gemm GMAC/s/SM', round(d['gemm_mac_per_s_per_sm']/1e9,1), 'wait', d['gemm_wait_share'])"
done
