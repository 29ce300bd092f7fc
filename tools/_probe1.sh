nproc; free -g; lscpu | head -20; df -h /tmp | tail -1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
