AB_CONFIGS=${AB_CONFIGS:-2} bash tools/ab.sh ${ROUNDS:-1} "$@" 2>&1 | tee gpurun_out/ab_${TAG:-x}.txt
