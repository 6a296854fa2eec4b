# r04g: k_bd_t phase trace (debug build on the box)
set -x
rm -rf build && GIST_EXTRA_NVCC_FLAGS=-DGIST_GEMM_TRACE python -m paper_2102_10424_b200.build > gpurun_out/r04g_build.log 2>&1; echo build=$?
GIST_GRAPH=0 python tools/bdt_trace.py > gpurun_out/r04g_trace.json 2> gpurun_out/r04g_trace.err; echo trace=$?
python tools/bdt_trace.py > gpurun_out/r04g_trace_graph.json 2>> gpurun_out/r04g_trace.err; echo trace2=$?
