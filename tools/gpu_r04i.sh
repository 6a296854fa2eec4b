# r04i: k_bd_t chunk-level trace (debug build)
set -x
rm -rf build && GIST_EXTRA_NVCC_FLAGS=-DGIST_GEMM_TRACE python -m paper_2102_10424_b200.build > gpurun_out/r04i_build.log 2>&1; echo build=$?
GIST_GRAPH=0 python tools/bdt_trace.py > gpurun_out/r04i_trace.json 2> gpurun_out/r04i_trace.err; echo trace=$?
