echo "== rows"; python tools/di_variants.py - build/variants/libgmt_b200_u4.so build/variants/libgmt_b200_u6.so build/variants/libgmt_b200_dyn3.so
echo "== views"; VIEWS=1 python tools/di_variants.py - build/variants/libgmt_b200_u4.so build/variants/libgmt_b200_u6.so build/variants/libgmt_b200_dyn3.so
