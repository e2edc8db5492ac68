# A/B of a variant library against the in-tree build on FSA configs 3/4 and
# the bench beam workload.  usage: tools/probes/ab_variant.sh <variant>
v=paper_2211_00484_b200/variants/librnntg_$1.so
for lib in "" "$v"; do  # in-tree = HEAD build
  echo "== ${lib:-in-tree} =="
  RNNTG_LIB=$lib python tools/prof_fsa.py 3 0 500 2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fsa3', round(d['decode_ms'],2), d['phase_share'])"
  RNNTG_LIB=$lib python tools/prof_fsa.py 4 0 500 2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fsa4', round(d['decode_ms'],2), d['phase_share'])"
  RNNTG_LIB=$lib python tools/prof_beam.py 1024 1000 2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('beam', d['decode_ms'])"
  RNNTG_LIB=$lib python tools/prof_beam.py 256 500 2 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('beam256', d['decode_ms'])"
done
