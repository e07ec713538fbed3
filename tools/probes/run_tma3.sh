cd tools/probes
for src in 1 0; do
./tma_stream 148 4 128 $src 1 0
./tma_stream 148 4 128 $src 2 0
./tma_stream 148 3 128 $src 3 0
./tma_stream 148 4 128 $src 2 1
./tma_stream 148 3 128 $src 3 1
./tma_stream 148 2 128 $src 6 1
./tma_stream 148 4 64 $src 4 1
done
