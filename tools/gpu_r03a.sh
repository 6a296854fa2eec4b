for bd in 1 0; do for sp in -1 0; do
GIST_BD=$bd GIST_SPMM_SPLIT=$sp python tools/heavy_dbg.py sage 24,600,40,5 bf16
GIST_BD=$bd GIST_SPMM_SPLIT=$sp python tools/heavy_dbg.py gcn 24,300,40,5 bf16
done; done
GIST_SPMM_SPLIT=0 python tools/heavy_dbg.py sage 24,300,40,5 fp32
python tools/heavy_dbg.py sage 24,300,40,5 fp32
