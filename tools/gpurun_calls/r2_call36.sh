# final-tree validation on 2 GPUs: smoke, full GPU suite (multi-GPU tests run at 2 ranks)
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/final4_smoke.log
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/final4_gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/final4_gpu_tests.log
