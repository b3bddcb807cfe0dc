set -x
python -m pytest tests -m gpu -x -q -s > gpurun_out/r2_gputests5.log 2>&1; tail -3 gpurun_out/r2_gputests5.log
PTYCHO_LIB=build/libptycho_no_v_step.so python -m pytest tests/test_gpu_fullsize.py -k "appp" -x -q -s > gpurun_out/r2_mutant_no_v_step.log 2>&1; tail -3 gpurun_out/r2_mutant_no_v_step.log
python bench.py --steps 2 --warmup 3 > gpurun_out/r2_bench5.json 2> gpurun_out/r2_bench5.err; tail -c 3000 gpurun_out/r2_bench5.err
bash tools/ab.sh build/libptycho_f2.so build/libptycho_f2_3stage.so > gpurun_out/r2_ab_3stage.txt 2>&1; cat gpurun_out/r2_ab_3stage.txt
