#!/bin/bash
# Records B200 box facts (device properties, topology, toolchain) into gpurun_out/boxfacts.txt
out=gpurun_out/boxfacts.txt
{
nvidia-smi
nvidia-smi topo -m
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,memory.total --format=csv
lscpu | head -20
nproc
python -c "
import torch
p=torch.cuda.get_device_properties(0)
print(p)
print('sms', p.multi_processor_count, 'l2', p.L2_cache_size, 'mem', p.total_memory)
print('nccl', torch.cuda.nccl.version())
"
} > $out 2>&1
echo done
