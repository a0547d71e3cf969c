# A/B of library builds by CUDA-event step time on config 2 (L2 flushed per step)
for lib in "$@"; do
  echo $lib $(EVOCA_B200_LIB=$PWD/paper_2406_09654_b200/$lib python tools/profile_step.py --steps 30 --time --flush 2>&1 | grep "step ms" | sed 's/.*best/best/')
done
