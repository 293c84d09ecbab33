mkdir -p gpurun_out/fcncu
for op in mlp3 2fcrelu; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fc_cluster -s 2 -c 1 -o gpurun_out/fcncu/$op -f python profiles/ncu_ops.py $op reps=4 > gpurun_out/fcncu/$op.log 2>&1
done
ls -la gpurun_out/fcncu
