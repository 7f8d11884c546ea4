export VK_FT_CAP=10
bash tools/variants_run.sh C4 20 2>&1 | grep config | cut -c1-40,118-150
echo C5; for c in 8 12 16 24 32; do VK_FT_CAP=$c timeout 300 python tools/stage_time.py C5 10 2>&1 | tail -1 | cut -c100-170; done
