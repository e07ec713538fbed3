cd tools/probes
for g in 0 1; do for iss in 1 2 4; do for st in 2 4; do ./tma_gather 148 $st $g $iss; done; done; done
./tma_gather 74 4 1 2; ./tma_gather 37 4 1 2
