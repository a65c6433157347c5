for o in "--maxrregcount=104" "--maxrregcount=112" "--maxrregcount=96"; do
 echo "== $o" >> gpurun_out/lg.txt
 BM_LGRAD_NVRTC_OPT="$o" timeout 300 python tools/cfg5_timeline_probe.py >> gpurun_out/lg.txt 2>&1
done
