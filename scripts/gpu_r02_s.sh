#!/bin/bash
# Round 2: multi-slab sketch at c4 with natural slab heights (reproduce the in-suite failures)
mkdir -p gpurun_out
MNB_TRACE=1 timeout 1200 python scripts/exp/slab_sweep.py c4 0,1024,1000,600,592,296,1184,1480 > gpurun_out/slab_sweep.log 2> gpurun_out/slab_sweep.err
