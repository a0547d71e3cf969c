# A/B of library builds (pass-1/pass-2 ncu durations on config 2) + GPU parity per variant
bash tools/gpu_ab2.sh "$@"
for l in "$@"; do echo $l; EVOCA_B200_LIB=$PWD/paper_2406_09654_b200/$l timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3; done
