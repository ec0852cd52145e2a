free -g; nproc; lscpu | grep -i "model name\|socket\|numa"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
