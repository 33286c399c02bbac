# host CPU and Keccak-f timing on the GPU box (the transcript's per-round cost)
O=gpurun_out/keccak; mkdir -p $O /tmp/kb
lscpu > $O/lscpu.txt
for f in "-O2" "-O3,-march=native"; do
  nvcc -std=c++17 -Xcompiler "$f" -Ipaper_2508_21393_b200/csrc -c paper_2508_21393_b200/csrc/transcript.cu -o /tmp/kb/t.o -gencode arch=compute_100a,code=sm_100a
  g++ -O2 tools/probes/keccak_bench.cpp /tmp/kb/t.o -o /tmp/kb/kb -L/usr/local/cuda/lib64 -lcudart
  for i in 1 2 3; do echo "$f: $(/tmp/kb/kb)"; done
done | tee $O/keccak.txt
grep -i "model name\|^CPU(s)" $O/lscpu.txt | cut -c1-120
