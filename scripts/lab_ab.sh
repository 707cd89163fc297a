# A/B probe set vs _old_tree: config 2, config 4, config-5 hidden at B=512
bash scripts/gpu_probe_us.sh
bash scripts/gpu_probe_us.sh 3072,8192,8192,8192,10 0.01 1024
bash scripts/gpu_probe_us.sh 3072,65536,65536,10 0.001 512
