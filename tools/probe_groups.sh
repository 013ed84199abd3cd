for g in 1 2 4; do timeout 300 python tools/group_probe.py 512 $g 4; done
for g in 1 2; do timeout 300 python tools/group_probe.py 64 $g 6; done
