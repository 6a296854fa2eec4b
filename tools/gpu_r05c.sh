# r05c: large-cluster BF16 case under each aggregation path
set -x
python tools/large_cluster_check.py > gpurun_out/r05c_lc.jsonl 2>&1
GIST_BDT_BUFS=1 python tools/large_cluster_check.py >> gpurun_out/r05c_lc.jsonl 2>&1
GIST_BD_T=0 python tools/large_cluster_check.py >> gpurun_out/r05c_lc.jsonl 2>&1
GIST_BD=0 python tools/large_cluster_check.py >> gpurun_out/r05c_lc.jsonl 2>&1
