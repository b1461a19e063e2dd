export PYTHONDONTWRITEBYTECODE=1
mkdir -p /tmp/ncu
run() { name=$1; shift; timeout 600 ncu --set full --clock-control none --import-source on -k regex:dbp_ -s 2 -c 1 -o /tmp/ncu/$name python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > /dev/null 2>&1; ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$name.csv 2>/dev/null; ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/raw_$name.csv 2>/dev/null; }
run e8192 --block-len 8192 --overlap 1400
