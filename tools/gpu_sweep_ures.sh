# mid-order isotropic shapes: CTA slots of the persistent u grid left free for the next chunk's w / v steps
for i in 8 9 10 12 14; do for r in 0 74 148 222; do python tools/grid_one.py $i 0 0 "P2S_LARGE_URESERVE=$r" | cut -c1-150; done; done
