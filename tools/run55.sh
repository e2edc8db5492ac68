# bulk-copied hypothesis state (sliced kernel) A/B + parity under the variant
RNNTG_LIB=paper_2211_00484_b200/variants/librnntg_bk1.so timeout 600 python -m pytest tests/test_gpu_sliced.py -q -x 2>&1 | tail -1
bash tools/run52.sh "$@"
