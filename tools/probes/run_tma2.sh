cd tools/probes
for src in 1 0; do
for br in 32 64 128 256; do ./tma_stream 148 4 $br $src 1; done
for is in 1 2 4; do ./tma_stream 148 4 128 $src $is; done
./tma_stream 148 3 256 $src 1
./tma_stream 148 2 256 $src 2
done
