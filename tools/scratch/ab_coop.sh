mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_coop.txt 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_coop.txt
for i in 1 2; do
for lib in ab/libmpxa_head.so paper_2309_07337_b200/libmpxa.so; do
  for emu in 0 4; do
    MPXA_LIB=$lib EMU=$emu ALGOS=pairwise,bruck,hier SIZES=16,4096,65536,1048576 timeout 300 python tools/lat_knobs.py 2>&1 | sed "s|^|$lib emu=$emu |" >> gpurun_out/ab_coop.txt
  done
done
done
cat gpurun_out/ab_coop.txt
