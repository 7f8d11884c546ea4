R=gpurun_out/s4e; mkdir -p $R
for g in "70,15,8" "75,13,7" "65,18,10" "78,12,6" "70,20,5"; do
  echo "guide $g"; VK_FT_GUIDE=$g timeout 300 python tools/stage_time.py C4 20 2>&1 | tail -1 | cut -c60-200
done
VK_FT_GUIDE="70,15,8" ncu --set full --import-source on --clock-control none -k regex:predict_fast_kernel -s 1 -c 1 -o $R/predict python tools/fit_profile_run.py C4 > $R/ncu_predict.log 2>&1; echo ncu rc=$?
