#!/bin/bash
# Round-2 evidence pass under gpurun: build, every GPU test, smoke, the default bench line and the
# reference arm, the other legs, the ncu launch list of the benched launch, a full capture of
# the throughput part.  usage: tools/r02_final.sh TAG
set -u
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
make -s all > $O/make.log 2>&1; echo "make rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2>&1; echo "c2 rc=$?"
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --config c3 --warm --no-cpu-baseline --no-e2e > $O/bench_c3seq.json 2>&1; echo "c3seq rc=$?"
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2>&1; echo "c5 rc=$?"
for p in 1 8; do timeout 600 python bench.py --config c4k --frames 1 --parts $p --no-cpu-baseline --no-e2e > $O/bench_c4k_p$p.json 2>&1; echo "c4k p$p rc=$?"; done
timeout 600 python bench.py --energy --no-cpu-baseline > $O/bench_energy.json 2>&1; echo "energy rc=$?"
timeout 600 python bench.py --prior --no-cpu-baseline > $O/bench_prior.json 2>&1; echo "prior rc=$?"
timeout 600 python bench.py --saliency --no-cpu-baseline > $O/bench_saliency.json 2>&1; echo "saliency rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 60 --csv --log-file $O/launches_c4_1024.csv $CMD > $O/ncu_launches.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve --launch-skip 1 -c 1 -o $O/prof_rest python tools/ncu_rest.py 256 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
