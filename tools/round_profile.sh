#!/bin/bash
# Round measurement set (one gpurun call): default bench line; apply / PCG-iteration / update_D launch lists
# under ncu, both cold-cache (ncu default: caches flushed before every kernel) and in-stream
# (--cache-control none: the L2 state the kernel really sees); level-1 SpMV per-warp timeline.
TAG=${1:-r02}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for CC in all none; do
  ncu --nvtx --nvtx-include "apply/" --metrics $M --cache-control $CC --clock-control none --csv \
      --log-file gpurun_out/${TAG}_apply_$CC.csv python tools/profile_apply.py 3 > /dev/null 2>&1
  python tools/launches.py gpurun_out/${TAG}_apply_$CC.csv > gpurun_out/${TAG}_apply_$CC.txt
  ncu --nvtx --nvtx-include "upd/" --metrics $M --cache-control $CC --clock-control none --csv \
      --log-file gpurun_out/${TAG}_upd_$CC.csv python tools/profile_update.py > /dev/null 2>&1
  python tools/launches.py gpurun_out/${TAG}_upd_$CC.csv > gpurun_out/${TAG}_upd_$CC.txt
done
AMGF_HOST_LOOP=1 ncu --nvtx --nvtx-include "pcg/" --metrics $M --clock-control none --csv \
    --log-file gpurun_out/${TAG}_pcg_all.csv python tools/profile_pcg_iter.py > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_pcg_all.csv > gpurun_out/${TAG}_pcg_all.txt
AMGF_SETUP_TIMING=1 python tools/time_update.py > gpurun_out/${TAG}_time_update.log 2>&1
python tools/time_apply.py 3 > gpurun_out/${TAG}_time_apply.jsonl 2>&1
tail -c 400 gpurun_out/${TAG}_bench.json; tail -1 gpurun_out/${TAG}_apply_none.txt
