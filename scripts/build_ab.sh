# build_ab.sh NAME "EXTRA NVCC FLAGS": an A/B variant of the library in build_ab/lib_NAME.so
set -e
NAME=$1; EXTRA=$2
D=/tmp/ab_$NAME
rm -rf $D; mkdir -p $D/csrc; cp -r paper_1806_09924_b200/csrc/* $D/csrc/; cp -r include $D/
sed -i "s#\.\./\.\./include#../include#g" $D/csrc/Makefile
sed -i "s#-I\.\./include#-I../include $EXTRA#" $D/csrc/Makefile
sed -i "s#OUT := \.\./libcrackfield_b200.so#OUT := ../lib.so#" $D/csrc/Makefile
rm -f $D/csrc/*.o
make -s -j8 -C $D/csrc
mkdir -p build_ab; cp $D/lib.so build_ab/lib_$NAME.so
