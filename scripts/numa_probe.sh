python -c "import torch; p=torch.cuda.get_device_properties(0); print(getattr(p, 'pci_bus_id', None)); import pynvml; pynvml.nvmlInit(); print(pynvml.nvmlDeviceGetCount())" > gpurun_out/numa.txt 2>&1
nvidia-smi topo -m >> gpurun_out/numa.txt 2>&1
for w in rmsnorm lora; do python bench.py --workload $w --no-verifier --no-cpu-baseline > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
python scripts/e2e_probe.py > gpurun_out/e2e.txt 2>&1
