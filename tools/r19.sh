timeout 60 tools/ubench/chunk_gemv > gpurun_out/ub_chunk.txt 2>&1; echo "chunk rc $?"
timeout 60 tools/ubench/fp64 > gpurun_out/ub_fp64.txt 2>&1; echo "fp64 rc $?"
PDG_ND_NODEP=1 PDG_ND_NOMATH=1 timeout 120 python tools/debug_nd.py 128 > gpurun_out/nd_nomath.log 2>&1; echo "nomath rc $?"
