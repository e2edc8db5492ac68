for r in 0 24 16 32; do RNNTG_DBG_FORCE_R=$r RNNTG_FUSED_PE=0 timeout 300 python tools/prof_beam.py 1024 1000 2 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($r, d['decode_ms'][-1], d['phase_share'], d['gemm_wait_share'])"; done
