for v in "BM_SYNC_SPIN_US=0" "X=1"; do
 echo "== $v" >> gpurun_out/spin.txt
 env $v timeout 300 python tools/cfg5_timeline_probe.py >> gpurun_out/spin.txt 2>&1
done
