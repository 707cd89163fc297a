#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
cat > /tmp/ncu_cfg2.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072,1024,512,10], density=0.01, batch_size=1024, lr=0.01))
data = smb.synthetic_dataset(seed=0, n_samples=8192, features=3072)
st = smb.FusedTrainStep(model, 1024, use_graph=False); st.attach_dataset(smb.DeviceDataset(data)); st.set_epoch(np.arange(8192))
for _ in range(4): st.step(0.01)
torch.cuda.synchronize()
PY
timeout 300 python /tmp/ncu_cfg2.py > gpurun_out/ncu_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python /tmp/ncu_cfg2.py > gpurun_out/ncu.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sddmm_pipe" -s 6 -c 1 -o gpurun_out/prof_cfg2_sddmm python /tmp/ncu_cfg2.py >> gpurun_out/ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu.log
tail -4 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | cut -c1-1500; tail -1 gpurun_out/ncu.log
