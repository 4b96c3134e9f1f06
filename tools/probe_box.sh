nvidia-smi; nproc; lscpu | grep -E 'Model name|^CPU\(s\)|Thread|Socket'; free -g | head -2
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p); print('L2', p.L2_cache_size, 'SMs', p.multi_processor_count)" 
