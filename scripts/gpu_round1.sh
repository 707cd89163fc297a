#!/bin/bash
# first GPU contact: kernel parity tests, smoke, scratch timings
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python scripts/time_step.py > gpurun_out/time_step.log 2>&1; echo "time exit $?" >> gpurun_out/time_step.log
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/time_step.log
# per-kernel device times (ncu launch list) of a short config-2 run
cat > /tmp/ncu_cfg2.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072,1024,512,10], density=0.01, batch_size=1024, lr=0.01))
data = smb.synthetic_dataset(seed=0, n_samples=8192, features=3072)
st = smb.FusedTrainStep(model, 1024, use_graph=False); st.attach_dataset(smb.DeviceDataset(data)); st.set_epoch(np.arange(8192))
for _ in range(4): st.step(0.01)
torch.cuda.synchronize()
PY
timeout 300 python /tmp/ncu_cfg2.py > gpurun_out/ncu_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"row_spmm|sddmm|softmax|gather|bias_rows" --csv --log-file gpurun_out/launches_cfg2.csv python /tmp/ncu_cfg2.py > gpurun_out/ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu.log
