# diagnostic timeline build: chunk landing vs chain probe starts (async load + iterate)
PTYCHO_LIB=build/libptycho_tl.so PTYCHO_AMP_TIMELINE=1 timeout 900 python tools/e2e_overlap.py > gpurun_out/timeline.log 2>&1
grep -m 40 TIMELINE gpurun_out/timeline.log
