AB_CONFIGS=2 bash tools/ab.sh 1 base nobar noload nostore nonl noio 2>&1 | tee gpurun_out/ab_ceilings_v9.txt
