cd /root/repo
for i in 1 2; do
for v in 0 1; do
  a=$(SGTK_SPMM_DC32=$v timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1)
  b=$(SGTK_SPMM_DC32=$v SGTK_PANEL_DEBUG=1 timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1)
  c=$(SGTK_SPMM_DC32=$v timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 128 2>&1 | tail -1)
  echo "dc32=$v | C3 $a | dense $b | d128 $c"
done; done
