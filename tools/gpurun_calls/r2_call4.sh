set -x
bash tools/ab.sh build/libptycho_f2.so build/libptycho_f2_3stage.so > gpurun_out/r2_ab_3stage.txt 2>&1
python tools/prof_chain.py --grid 1x1 --probes 1 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 150 -c 1 -o gpurun_out/r2_bwd_lone_f2 python tools/prof_chain.py --grid 1x1 --probes 1 > gpurun_out/r2_ncu_lone.log 2>&1
python -m pytest tests/test_gpu_fullsize.py -k "appp or lt_small-5" -x -q -s > gpurun_out/r2_fullsize.log 2>&1
PTYCHO_LIB=build/libptycho_no_v_step.so python -m pytest tests/test_gpu_fullsize.py -k "appp" -x -q -s > gpurun_out/r2_mutant_no_v_step.log 2>&1
python -m pytest tests/test_gpu_recon_large.py -x -q -s > gpurun_out/r2_recon_large.log 2>&1
tail -2 gpurun_out/r2_fullsize.log gpurun_out/r2_mutant_no_v_step.log gpurun_out/r2_recon_large.log
cat gpurun_out/r2_ab_3stage.txt
