#!/bin/bash
# Round measurement (profiles/rNN, collected by scripts/collect_profiles.sh): gpu tests, smoke, bench lines (c3 default + per-candidate A/B,
# c2, c4, c5, reference arm), launch lists (c3, c4), ncu --set full of the dominant kernels.
cd $GRAFT_REPO_ROOT
T=${1:-r1d}
O=gpurun_out/$T
mkdir -p $O
python -c "import oracle; oracle.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --per-candidate --no-cpu-baseline > $O/bench_c3_per_candidate.json 2> $O/bench_c3_pc.err; echo "c3 pc rc=$?"
timeout 900 python bench.py --config c2 > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c4 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --config c5 > $O/bench_c5.json 2> $O/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --f3 > $O/bench_c3_f3.json 2> $O/bench_c3_f3.err; echo "c3 f3 rc=$?"
timeout 900 python scripts/f1_sweep.py --f4 --out $O/f1_sweep.json > $O/f1_sweep.log 2>&1; echo "f1 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_c3.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1; echo "launches c3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1; echo "launches c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_exh_(memo|bp)" -c 2 -o $O/full_c3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_exhaustive" -c 1 -o $O/full_c3_pc python bench.py --per-candidate --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/ncu_c3_pc.log 2>&1; echo "ncu c3 pc rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_allocate" -c 5 -o $O/full_c4_alloc python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/ncu_c4a.log 2>&1; echo "ncu c4 alloc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_generate" -c 1 -o $O/full_c4_gen python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/ncu_c4g.log 2>&1; echo "ncu c4 gen rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_allocate" -c 5 -o $O/full_c3_alloc python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-direct > $O/ncu_c3a.log 2>&1; echo "ncu c3 alloc rc=$?"
# summarise the ncu reports here and drop them (gpurun returns at most 64 MiB)
for r in full_c3:ncu_full_bitsliced_c3:c3_exhaustive_20sm:69475500000 \
         full_c3_alloc:ncu_full_k_allocate_c3:c3_exhaustive_20sm_allocate: \
         full_c3_pc:ncu_full_per_candidate_c3:c3_exhaustive_20sm_per_candidate:69475500000 \
         full_c4_alloc:ncu_full_k_allocate_c4:c4_b200_148sm_allocate: \
         full_c4_gen:ncu_full_k_generate_c4:c4_b200_148sm_generate: ; do
  IFS=: read rep txt key cand <<< "$r"
  [ -f $O/$rep.ncu-rep ] || continue
  python scripts/ncu_summary.py $O/$rep.ncu-rep --top 14 > $O/$txt.txt
  python scripts/ncu_metrics.py $O/$rep.ncu-rep $key --out $O/ncu_metrics.json ${cand:+--candidates $cand} \
    --note "ncu --set full --clock-control none at the bench's launch configuration (scripts/gpu_round.sh $T); dram_bytes per call, cold L2" > /dev/null
done
[ "$KEEP_REPORTS" = "c3" ] && mv $O/full_c3.ncu-rep $O/keep_full_c3.ncu-rep
rm -f $O/*.ncu-rep
[ -f $O/keep_full_c3.ncu-rep ] && mv $O/keep_full_c3.ncu-rep $O/full_c3.ncu-rep
# compute-sanitizer is closed on the GPU pool (it left GPUs needing a reset): no sanitizer pass
# bash scripts/gpu_sanitize.sh $T
ls $O; du -sh $O
