# row-split CTA size (diag OZMM_ROW_CTA: threads per CTA of the cluster row kernel; 1024 = one CTA per row)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/cols_probe.py --row-variants "c128:OZMM_ROW_CTA=128,c256:OZMM_ROW_CTA=256,c512:OZMM_ROW_CTA=512,c1024:OZMM_ROW_CTA=1024"
python tools/cols_probe.py --n 8192 --p 8192 --row-variants "c128:OZMM_ROW_CTA=128,c256:OZMM_ROW_CTA=256,c512:OZMM_ROW_CTA=512,c1024:OZMM_ROW_CTA=1024"
cp /tmp/rel.so $L
