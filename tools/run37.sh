timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for gc in 0 1; do RNNTG_GREEDY_CLUSTER=$gc timeout 600 python tools/perf_configs.py 2>&1 | grep -E "config1" | cut -c1-160; done
