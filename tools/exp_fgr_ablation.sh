set -x
V=paper_2510_26180_b200/lib/variants
python tools/tune_c4.py 131072 jsweep 2>&1 | grep -v Warn
for pad in 15168 34624 89920; do KLE_FGR_PAD_SMEM=$pad python tools/tune_c4.py 131072 2>&1 | tail -1; done
for e in 1 2 3; do KLE_B200_LIB=$V/libkle_exp$e.so python tools/tune_c4.py 131072 2>&1 | tail -1; KLE_FGR_PAD_SMEM=34624 KLE_B200_LIB=$V/libkle_exp$e.so python tools/tune_c4.py 131072 2>&1 | tail -1; done
