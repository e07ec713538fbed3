cd tools/probes
for src in 0 1; do
for ctas in 1 8 37 74 148; do ./tma_stream $ctas 4 128 $src; done
for st in 2 4 6 8 12; do ./tma_stream 148 $st 64 $src; done
for st in 2 3 4 5 6; do ./tma_stream 148 $st 128 $src; done
done
