nproc; lscpu | grep -E "Model name|Socket|Thread|Core"; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "
import torch
p=torch.cuda.get_device_properties(0)
print(p)
print('L2', p.L2_cache_size, 'SMs', p.multi_processor_count, 'smem/block optin', getattr(p,'shared_memory_per_block_optin',None), 'smem/SM', getattr(p,'shared_memory_per_multiprocessor',None), 'regs/SM', getattr(p,'regs_per_multiprocessor',None), 'max threads/SM', p.max_threads_per_multi_processor)
"
