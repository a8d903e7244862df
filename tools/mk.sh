#!/bin/bash
# build libp2s_b200.so (absolute paths; prints the tail of any failure)
make -C /root/repo/paper_1703_09619_b200/csrc -s -j8 > /tmp/mk.log 2>&1 || { tail -30 /tmp/mk.log; exit 1; }
ls -la --time-style=+%T /root/repo/paper_1703_09619_b200/libp2s_b200.so
