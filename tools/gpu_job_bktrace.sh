export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
for c in 1 2 9 16; do R1_BK_TRACE=$c REPS=1 python tools/bk_time_probe.py 6500 2>&1 | grep 'r1 bk'; done
for c in 1 4; do R1_BK_TRACE=$c REPS=1 python tools/bk_time_probe.py 1000 2>&1 | grep 'r1 bk'; done
