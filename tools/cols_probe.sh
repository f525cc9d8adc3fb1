# column-split variants (diag build), C3 and C2 shapes
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/cols_probe.py
python tools/cols_probe.py --n 8192 --p 8192
python tools/cols_probe.py --n 1000 --p 777 --k 12
cp /tmp/rel.so $L
