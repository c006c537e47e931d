for v in poly1 poly2; do echo "parity $v"; LSK_LIB_PATH=scripts/variants/liblsk_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "implicit" 2>&1 | tail -2; done
AB_C5=1 AB_C1=1 bash scripts/gpu_runs/gpu_ab.sh base poly1 poly2
