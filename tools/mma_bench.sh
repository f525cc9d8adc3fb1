# tools/mma_bench.cu sweep: cycles per MMA of the pair issue loop against the 64-cycle floor
set -u
B=./tools/mma_bench
# args: rounds prods commit wait nacc run fill nbars N grid mode
echo "# mode 0 (runtime loop with % ops): run 4 vs 8"
$B 1000 8 0 0 4 4 1 5 128 148 0
$B 1000 8 0 0 4 8 1 5 128 148 0
echo "# mode 1 (param-space info words, like the pair kernel): prods per round, commit+wait"
for prods in 2 4 8 16; do $B $((16000/prods/4)) $prods 0 0 4 4 1 5 128 148 1; done
for prods in 2 4 8 16; do $B $((16000/prods/4)) $prods 1 1 4 4 1 5 128 148 1; done
echo "# mode 2 (compile-time 8 products, new acc + new B each), 3 (same acc), 4 (same B)"
for m in 2 3 4; do $B 500 8 0 0 4 4 1 5 128 148 $m; $B 500 8 1 1 4 4 1 5 128 148 $m; done
$B 500 8 0 0 4 4 0 5 128 148 2
