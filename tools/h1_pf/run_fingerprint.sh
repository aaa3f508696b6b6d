#!/bin/bash
# Which kind of host is this box?  CPU model/stepping/MHz/cache + H1 alone and next to DMA + the DMA alone
cd "$(dirname "$0")" && make -s
grep -m1 -E "^model\s" /proc/cpuinfo; grep -m1 stepping /proc/cpuinfo; grep -m1 "cpu MHz" /proc/cpuinfo
grep -m1 -o -E "amx_tile|avx512_fp16|avx_vnni" /proc/cpuinfo | sort -u | tr '\n' ' '; echo
lscpu | grep -E "L2 cache|L3 cache|BogoMIPS"
free -g | head -2
./h1_pf 16 1e8 4 0 pwdyn1024 pwdyn1024
./h1_pf 16 1e8 4 1 idle pwdyn1024 pwdyn1024
./h1_pf 8 1e8 4 0 pwdyn1024
