set -x
uname -m; nproc; lscpu | head -25; free -g; nvidia-smi -L; nvidia-smi topo -m; ls /root/reference 2>&1 | head -3
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.limit --format=csv
./tools/ubench_ops
./tools/ubench_ops
