set -x
rm -f gpurun_out/pdl_ab.log
for cfg in "0 1" "2 1" "3 1" "7 1" "3 0" "7 0" "1 0"; do
  set -- $cfg
  for wl in "A3 --batch 8" "A4 --batch 8" "A1 --batch 1"; do
    echo "PDL=$1 QTRIG=$2" >> gpurun_out/pdl_ab.log
    QFLASH_PDL=$1 QFLASH_PDL_QTRIG=$2 timeout 300 python tools/graph_ab.py --workload $wl 2>&1 | grep graph | tee -a gpurun_out/pdl_ab.log
  done
done
