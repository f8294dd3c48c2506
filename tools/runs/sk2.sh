cd /root/repo
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sk_launch.csv python bench.py --no-cpu --workload cora-gcn --steps 1 --warmup 3 > /dev/null 2>&1; echo "rc $?"
