set -x
timeout 300 python -m pytest tests/test_gpu_gat.py -q -x -k "one_step and bf16 and ragged" > gpurun_out/r02v_new.log 2>&1; echo new=$?
cp paper_2102_10424_b200/csrc/gat.cu /tmp/gat_new.cu
cp tools/gat_head.cu.txt paper_2102_10424_b200/csrc/gat.cu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02v_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_gat.py -q -x -k "one_step and bf16 and ragged" > gpurun_out/r02v_head.log 2>&1; echo head=$?
