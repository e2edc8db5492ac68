# joiner GEMM tiling threshold (RNNTG_BAL_MIN_R builds) across batch sizes
for v in "$@"; do
for bt in "128 500" "256 500" "512 500" "1024 300"; do set -- $bt
RNNTG_LIB=paper_2211_00484_b200/variants/librnntg_$v.so RNNTG_SLICED=1 timeout 300 python tools/prof_beam.py $1 $2 3 | python -c "import json,sys;d=json.load(sys.stdin);print('$v B=$1 T=$2', round(min(d['decode_ms']),2), 'phase', d['phase_share'], d['checksum'])"
done; done
