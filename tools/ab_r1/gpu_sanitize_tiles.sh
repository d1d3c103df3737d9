for T in memcheck racecheck synccheck; do
  echo "== $T"
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_tiles.py > gpurun_out/san_tiles_$T.txt 2>&1
  grep -E "SUMMARY|loss|rror" gpurun_out/san_tiles_$T.txt | head -40
done
