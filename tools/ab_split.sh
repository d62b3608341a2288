for lib in reg cpasync; do for sp in 1 512 1024 4096; do
  echo "=== $lib split $sp"
  SLPA_LIB=build_ab/libslpa_$lib.so SLPA_HI_SPLIT=$sp python tools/prof_run.py --scale 24 --runs 2 | tail -1
done; done
for lib in reg cpasync; do echo "=== $lib async"; SLPA_LIB=build_ab/libslpa_$lib.so python tools/prof_run.py --scale 24 --runs 2 --mode async | tail -1; done
