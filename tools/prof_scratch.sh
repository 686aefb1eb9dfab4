V=paper_2008_03095_b200/lib/variants
for t in base new base new; do lib=$V/libinfuser_b200_$t.so; [ $t = new ] && lib=paper_2008_03095_b200/lib/libinfuser_b200.so; echo $t; INFUSER_B200_LIB=$lib python tools/profile_e2e.py c2 --pinned 2>&1 | head -2 | cut -c 1-330; done
