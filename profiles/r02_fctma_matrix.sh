OUT=gpurun_out/fctma; mkdir -p $OUT
timeout 900 python profiles/fctma_matrix.py > $OUT/matrix.txt 2>&1
cat $OUT/matrix.txt
