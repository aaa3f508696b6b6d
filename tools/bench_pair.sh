#!/bin/bash
# Both bench arms the way the driver runs them (reference first), N=1.
mkdir -p gpurun_out
STEPS=${STEPS:-20}; WARM=${WARM:-5}; TAG=${TAG:-r02}
python bench.py --impl reference --gpus 1 --steps $STEPS --warmup $WARM > gpurun_out/${TAG}_ref.out 2> gpurun_out/${TAG}_ref.err
python bench.py --gpus 1 --steps $STEPS --warmup $WARM ${EXTRA:-} > gpurun_out/${TAG}_b200.out 2> gpurun_out/${TAG}_b200.err
tail -c 3000 gpurun_out/${TAG}_b200.err
