for i in 1 2; do
PF_REC_LAYOUT=hc3 WL="hd4 uhd4" REPS=1 bash tools/bench_variants.sh base
PF_REC_LAYOUT=split WL="hd4 uhd4" REPS=1 bash tools/bench_variants.sh split
done
