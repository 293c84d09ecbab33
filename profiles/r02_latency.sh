#!/bin/bash
# r02: the paper's latency protocol from C++ through the C ABI (tcb latency)
OUT=gpurun_out/r02_latency; mkdir -p $OUT
T=paper_1802_04730_b200/bin/tcb; F=paper_1802_04730_b200/tc/ops.tc
{
$T latency $F --def tmm --sizes M=128,N=256,K=32
$T latency $F --def tmm --sizes M=128,N=1024,K=1024
$T latency $F --def tbmm --sizes B=500,N=26,M=72,K=26
$T latency $F --def MLP1 --sizes B=128,M=1128,O=128,N=1128
$T latency $F --def 2FCRelu --sizes B=128,M=1128,O=128,N=1128,P=64
$T latency $F --def MLP3 --sizes B=128,M=128,O=64,N=128,P=32,Q=2,O1__0=128,O1__1=128
$T latency $F --def C3 --sizes B=128,WX=1024,WY=1000
$T latency $F --def 3KRU --sizes D0=32,N0=16,D1=32,N1=16,D2=32,N2=16,M=256
$T latency $F --def tmm --sizes M=128,N=256,K=32 --math 3xtf32
} > $OUT/latency.jsonl 2> $OUT/latency.err
cat $OUT/latency.jsonl $OUT/latency.err
