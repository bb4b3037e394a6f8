# Build recipe for the B200 fused-LCE operator, its C oracle and the
# reference-built checker.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same targets.
NVCC      ?= nvcc
CXX       := /usr/bin/g++
CC        := /usr/bin/gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
             --expt-relaxed-constexpr -diag-suppress 177
REF_DIR   ?= /root/reference/proj

PKG       := paper_2511_17599_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libfce.so
ORACLE    := oracle/liboracle.so
REF_LIB   := oracle/_ref/libfce_ref.so

DROPIN_TEST := tests/cpp/test_dropin
DROPIN_BENCH := tests/cpp/bench_dropin

all: $(LIB) $(ORACLE) ref $(DROPIN_TEST) $(DROPIN_BENCH)

# C++ drop-in API (include/fusedce) against the oracle; runs on a B200
$(DROPIN_TEST): tests/cpp/test_dropin.cpp $(wildcard include/fusedce/*.hpp include/fusedce/detail/*.hpp) \
                include/fce/fce.h $(LIB) $(ORACLE)
	$(CXX) -std=c++20 -O2 -Iinclude -I/usr/local/cuda/include -o $@ tests/cpp/test_dropin.cpp \
	    -L$(PKG) -lfce -Loracle -loracle -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,'$$ORIGIN/../../oracle' -Wl,-rpath,/usr/local/cuda/lib64

$(DROPIN_BENCH): tests/cpp/bench_dropin.cpp $(wildcard include/fusedce/*.hpp include/fusedce/detail/*.hpp) \
                 include/fce/fce.h $(LIB)
	$(CXX) -std=c++20 -O2 -Iinclude -I/usr/local/cuda/include -o $@ tests/cpp/bench_dropin.cpp \
	    -L$(PKG) -lfce -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

$(LIB): $(CSRC)/fce_kernels.cu $(CSRC)/fce_bwd.cu $(CSRC)/fce_pair.cu $(CSRC)/fce_fwd_pair.cu $(CSRC)/fce_api.cpp $(CSRC)/fce_vp.cpp $(CSRC)/fce_internal.h \
        $(CSRC)/fce_comm.cpp $(CSRC)/fce_comm.cu $(CSRC)/fce_comm.h include/fce/fce_vp.h \
        $(CSRC)/sm100_ptx.cuh include/fce/fce.h
	$(NVCC) $(NVFLAGS) -shared -cudart static -o $@ $(CSRC)/fce_kernels.cu $(CSRC)/fce_bwd.cu $(CSRC)/fce_pair.cu $(CSRC)/fce_fwd_pair.cu $(CSRC)/fce_api.cpp \
	    $(CSRC)/fce_vp.cpp $(CSRC)/fce_comm.cpp $(CSRC)/fce_comm.cu -ldl -lpthread -lrt

$(ORACLE): oracle/fce_oracle.c oracle/fce_oracle.h
	$(CC) -O2 -std=c11 -fPIC -shared -fopenmp -ffp-contract=off -o $@ oracle/fce_oracle.c -lm

# The reference itself, compiled in place from /root/reference (header-only
# C++20) through a thin extern "C" shim; output stays in oracle/_ref/.
ref:
	@if [ -d "$(REF_DIR)/include/fusedce" ]; then $(MAKE) $(REF_LIB); \
	 else echo "reference tree absent: using prebuilt $(REF_LIB) if present"; fi

$(REF_LIB): oracle/ref_shim.cpp
	mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O3 -march=x86-64-v3 -fPIC -shared -pthread -Dfusedce=fusedce_ref -ffp-contract=off \
	    -I$(REF_DIR)/include -o $@ oracle/ref_shim.cpp

clean:
	rm -f $(LIB) $(ORACLE) $(REF_LIB) $(DROPIN_TEST) $(DROPIN_BENCH)

.PHONY: all ref clean
