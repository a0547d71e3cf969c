# A/B of library builds: CUDA-event step time of a config.  usage: gpu_ab_libs.sh CONFIG LIB...
cfg=$1; shift
for i in 1 2; do
for lib in "$@"; do
  echo $lib $(EVOCA_B200_LIB=$PWD/paper_2406_09654_b200/$lib python tools/profile_step.py --config $cfg --steps 8 --flush --time 2>/dev/null | head -1)
done; done
