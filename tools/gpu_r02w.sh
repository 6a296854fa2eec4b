for m in f r c; do GIST_GAT_HALF=$m timeout 300 python -m pytest tests/test_gpu_gat.py -q -x -k "one_step and bf16 and ragged" > gpurun_out/r02w_$m.log 2>&1; echo $m=$?; done
