set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_hve.py tests/test_gpu_stash_free.py -x -q > gpurun_out/r2_tma_tests.log 2>&1; tail -3 gpurun_out/r2_tma_tests.log
python -m pytest tests/test_gpu_fullsize.py -k "appp or lt_small-5" -x -q -s > gpurun_out/r2_tma_fullsize.log 2>&1; tail -3 gpurun_out/r2_tma_fullsize.log
PTYCHO_LIB=build/libptycho_no_v_step.so python -m pytest tests/test_gpu_fullsize.py -k "appp" -x -q -s > gpurun_out/r2_tma_mutant.log 2>&1; tail -3 gpurun_out/r2_tma_mutant.log
bash tools/ab.sh build/libptycho_tma.so build/libptycho_notma.so build/libptycho_f2.so > gpurun_out/r2_ab_tma.txt 2>&1; cat gpurun_out/r2_ab_tma.txt
