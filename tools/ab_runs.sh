for i in 1 2 3; do
  PF_NO_TILES=1 WL="hd4 uhd4" REPS=1 bash tools/bench_variants.sh base | sed 's/^/notile /'
  WL="hd4 uhd4" REPS=1 bash tools/bench_variants.sh base | sed 's/^/tiles  /'
done
