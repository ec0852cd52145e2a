#!/bin/bash
# Round-end verification on one B200: GPU tests, smoke, bench lines (own arm,
# reference arm, config 5), config 1 / config 3 drivers, the gloo-staged
# world-2 bench validation and the bench launch list under ncu.
mkdir -p gpurun_out/final
O=gpurun_out/final
(timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5) > $O/tests.log
timeout 180 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err
timeout 400 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python profiles/run_cg1.py > $O/cg1.json 2> $O/cg1.err
MODELS=b200 timeout 600 python profiles/run_config3.py > $O/c3_b200.json 2> $O/c3_b200.err
timeout 600 python profiles/run_config3.py > $O/c3_shipped.json 2> $O/c3_shipped.err
SPMVTUNE_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_n2_gloo.json 2> $O/bench_n2_gloo.err
timeout 900 python bench.py --workload config5 --steps 2 --warmup 3 > $O/config5.json 2> $O/config5.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches.csv python profiles/run_solve.py > $O/ncu_run.log 2>&1
cat $O/tests.log $O/smoke.log | tail -4
for f in bench bench_ref cg1 c3_b200 c3_shipped bench_n2_gloo config5; do echo "== $f"; tail -c 400 $O/$f.json; echo; done
