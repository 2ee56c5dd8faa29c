set -u
O=gpurun_out; mkdir -p $O
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('persisting max', getattr(p,'persisting_l2_cache_max_size',None), 'L2', p.L2_cache_size)"
for r in 1 2; do
for v in 0 1; do
LCC_L2PERSIST=$v timeout 300 python bench.py --no-cpu --no-e2e > $O/b.json 2>/dev/null; echo "l2p=$v $(python -c "import json;d=json.load(open('$O/b.json'));print(round(d['value'],3), round(d['roofline']['kernel_ms_per_step'],3))")"
done; done
