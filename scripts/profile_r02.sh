#!/bin/bash
# Round-2 evidence in one GPU call: bench line, reference arm, launch list of one
# n=300 solve, per-launch DRAM traffic of the containment / expansion / dedupe
# kernels, full ncu captures of the largest existence-query and marking launches.
# Outputs under gpurun_out/r02/.
set -x
cd "$(dirname "$0")/.."
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
tail -c 3000 $O/bench.json
python bench.py --impl reference --steps 2 --warmup 1 --no-ref-full > $O/bench_reference.json 2> $O/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python scripts/one_solve.py random:300,2,0 44 > /dev/null 2>&1
python scripts/launch_summary.py $O/launches.csv 30 > $O/launches.txt
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"contain_pool|trie_pool" --csv --log-file $O/traffic_contain.csv \
    python scripts/one_solve.py random:300,2,0 44 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"expand_sliced|dd_single" --csv --log-file $O/traffic_micro.csv \
    python scripts/micro_ab.py random:300,2,0 > /dev/null 2>&1
python scripts/traffic_summary.py $O/dram_traffic.json $O/traffic_contain.csv $O/traffic_micro.csv
# full captures of the last (largest) existence query and marking launch of one solve
NE=$(grep -c "trie_pool_kernel<5, 0, 1>" $O/launches.csv)
NM=$(grep -c "contain_pool_kernel<5, 1, 0>" $O/launches.csv)
ncu --set full --import-source on --clock-control none -k regex:"trie_pool_kernel" \
    --launch-skip $((NE - 1)) --launch-count 1 -o $O/ncu_trie_exist \
    python scripts/one_solve.py random:300,2,0 44 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"contain_pool_kernel" \
    --launch-skip $((NM - 1)) --launch-count 1 -o $O/ncu_contain_mark \
    python scripts/one_solve.py random:300,2,0 44 > /dev/null 2>&1
# north-star kernels at HBM scale (2^24 parents / rows, n=300): one launch each
for m in img pre dedupe; do
  K=expand_sliced; [ $m = dedupe ] && K=dd_single
  ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip 1 --launch-count 1 \
      -o $O/ncu_micro_$m python scripts/micro_one.py $m > /dev/null 2>&1
done
for r in ncu_trie_exist ncu_contain_mark ncu_micro_img ncu_micro_pre ncu_micro_dedupe; do
  python scripts/ncu_summary.py $O/$r.ncu-rep > $O/$r.txt
done
python scripts/baselines.py $O/baselines.json --skip-full > $O/baselines.log 2>&1
gzip -f $O/launches.csv $O/traffic_contain.csv $O/traffic_micro.csv
rm -f $O/*.ncu-rep  # summaries kept (gpurun copies back at most 64 MiB)
ls -la $O
