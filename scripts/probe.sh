nvidia-smi > gpurun_out/probe_smi.txt 2>&1
nproc > gpurun_out/probe_cpu.txt; lscpu >> gpurun_out/probe_cpu.txt; free -g >> gpurun_out/probe_cpu.txt
python -c "
import torch
p=torch.cuda.get_device_properties(0)
print(p)
print('L2', p.L2_cache_size, 'sms', p.multi_processor_count)
" > gpurun_out/probe_torch.txt 2>&1
