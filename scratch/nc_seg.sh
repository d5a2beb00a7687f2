#!/bin/bash
for P in 3 4 7 9 16 37; do echo -n "bwd P2=$P "; LA_FULL_SEGMENTS=$P python scratch/nc_prof.py | tail -1; done
for P in 5 7 9 16 37; do echo -n "fwd P2=$P "; LA_FULL_SEGMENTS_F=$P python scratch/nc_prof.py | tail -1; done
