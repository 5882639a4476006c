#!/bin/bash
# Copy one gpu_round.sh run (gpurun_out/TAG) into profiles/OUT: bench lines, pytest / smoke
# logs, launch lists (csv + per-kernel shares), ncu --set full summaries, ncu_metrics.json.
#   bash scripts/collect_profiles.sh r02a r02
set -e
T=$1; O=profiles/$2; I=gpurun_out/$T
mkdir -p $O
for f in bench_c2.json bench_c3.json bench_c3_per_candidate.json bench_c4.json bench_c5.json \
         bench_c3_f3.json bench_reference_c3.json pytest_gpu.log smoke.log launches_c3.csv \
         launches_c4.csv f1_sweep.json f1_sweep.log; do
  [ -f $I/$f ] && cp $I/$f $O/
done
for l in c3 c4; do
  [ -f $I/launches_$l.csv ] && python scripts/ncu_summary.py --launches $I/launches_$l.csv > $O/launches_$l.txt
done
S=$(python -c "import gp_workloads as W; print(10*10000)")
for r in full_c3:ncu_full_bitsliced_c3:c3_exhaustive_20sm:69475500000 \
         full_c3_alloc:ncu_full_k_allocate_c3:c3_exhaustive_20sm_allocate: \
         full_c3_pc:ncu_full_per_candidate_c3:c3_exhaustive_20sm_per_candidate:69475500000 \
         full_c4_alloc:ncu_full_k_allocate_c4:c4_b200_148sm_allocate: \
         full_c4_gen:ncu_full_k_generate_c4:c4_b200_148sm_generate: ; do
  IFS=: read rep txt key cand <<< "$r"
  if [ -f $I/$rep.ncu-rep ]; then
    python scripts/ncu_summary.py $I/$rep.ncu-rep --top 14 > $O/$txt.txt
    python scripts/ncu_metrics.py $I/$rep.ncu-rep $key --out $O/ncu_metrics.json \
      ${cand:+--candidates $cand} --note "ncu --set full --clock-control none at the bench's launch configuration (scripts/gpu_round.sh $T); dram_bytes per call, cold L2" > /dev/null
  elif [ -f $I/$txt.txt ]; then  # summarised on the GPU box (reports exceed gpurun's 64 MiB)
    cp $I/$txt.txt $O/
  fi
done
[ -f $I/ncu_metrics.json ] && [ ! -f $O/ncu_metrics.json ] && cp $I/ncu_metrics.json $O/
for f in compute_sanitizer_memcheck.log compute_sanitizer_racecheck.log compute_sanitizer_synccheck.log; do
  [ -f $I/$f ] && cp $I/$f $O/
done
ls $O
