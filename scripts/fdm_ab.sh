#!/bin/bash
# A/B of the d = 3 element-block preconditioner (device time, CUDA graph):
# fdm3_kernel with parameter factors (default), with shared-memory factors
# (STG_FDM3_SMEMC=1), and the two-half kernel (STG_FDM_V1=1).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
python scripts/fdm_graph_bench.py c4 > gpurun_out/fdm_ab_param.json 2>&1
STG_FDM3_SMEMC=1 python scripts/fdm_graph_bench.py c4 > gpurun_out/fdm_ab_smemc.json 2>&1
STG_FDM_V1=1 python scripts/fdm_graph_bench.py c4 > gpurun_out/fdm_ab_v1.json 2>&1
python scripts/fdm_graph_bench.py c4 1 > gpurun_out/fdm_ab_tblock.json 2>&1
python scripts/fdm_graph_bench.py c2 > gpurun_out/fdm_ab_c2_fdm2.json 2>&1
STG_NO_FDM2=1 python scripts/fdm_graph_bench.py c2 > gpurun_out/fdm_ab_c2_dense.json 2>&1
