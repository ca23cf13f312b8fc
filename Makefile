# Builds the product library (sm_100a CUDA kernels + C-ABI host runtime) in-tree:
#   paper_2211_14969_b200/_lib/libhps_leaf_b200.so
# and the CPU oracle (test infrastructure) via oracle/Makefile.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -Iinclude \
             -Ipaper_2211_14969_b200/csrc -Xptxas -v $(EXTRA)
SRC       := paper_2211_14969_b200/csrc
OBJDIR    := build/obj
LIB       := paper_2211_14969_b200/_lib/libhps_leaf_b200.so
CU        := $(SRC)/k0_fields.cu $(SRC)/k1_assemble.cu $(SRC)/k1_operator.cu $(SRC)/k2s_small.cu $(SRC)/k4_scatter.cu $(SRC)/k5_leaf_solve.cu $(SRC)/k6_residual.cu $(SRC)/k7_reconstruct.cu $(SRC)/k9_fp64_peak.cu
CPP       := $(SRC)/hps_host.cpp $(SRC)/hps_api.cpp
HDRS      := $(wildcard $(SRC)/*.h $(SRC)/*.cuh include/*.h include/hps/*.hpp)
# K2/K3 are built twice: 8-warp CTAs (g256) and 4-warp CTAs for small leaves (g128).
K2OBJS    := $(OBJDIR)/k2_g256.o $(OBJDIR)/k2_g128.o
# K2 tuning knobs (CTAs/SM, cp.async pipeline stages, K chunk); `make variant` builds A/B copies.
G256_NSTAGE ?= 3
G256_KC     ?= 16
G128_CTAS   ?= 4
G128_NSTAGE ?= 2
G128_KC     ?= 16
OBJS      := $(patsubst $(SRC)/%,$(OBJDIR)/%.o,$(CU) $(CPP)) $(K2OBJS)

SLIB      := paper_2211_14969_b200/_lib/libhps_slablu_b200.so

all: $(LIB) $(SLIB) oracle

$(OBJDIR)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $(OBJDIR)/$*.ptxas.log 2>&1 || (cat $(OBJDIR)/$*.ptxas.log; exit 1)

$(OBJDIR)/k2_g256.o: $(SRC)/k2_lu_schur.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -DHPS_NT=256 -DHPS_CFG=g256 -DHPS_CTAS=2 -DHPS_NSTAGE=$(G256_NSTAGE) -DHPS_KC=$(G256_KC) -DHPS_MAX_ROWS=2048 \
	    -c $< -o $@ > $(OBJDIR)/k2_g256.ptxas.log 2>&1 || (cat $(OBJDIR)/k2_g256.ptxas.log; exit 1)

$(OBJDIR)/k2_g128.o: $(SRC)/k2_lu_schur.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -DHPS_NT=128 -DHPS_CFG=g128 -DHPS_CTAS=$(G128_CTAS) -DHPS_NSTAGE=$(G128_NSTAGE) -DHPS_KC=$(G128_KC) -DHPS_MAX_ROWS=640 \
	    -c $< -o $@ > $(OBJDIR)/k2_g128.ptxas.log 2>&1 || (cat $(OBJDIR)/k2_g128.ptxas.log; exit 1)

$(OBJDIR)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

# GPU SlabLU: its own library, cuSOLVER/cuBLAS for the dense blocks.
$(OBJDIR)/slablu.o: $(SRC)/slablu.cu include/hps_slablu.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $(OBJDIR)/slablu.ptxas.log 2>&1 || (cat $(OBJDIR)/slablu.ptxas.log; exit 1)

$(SLIB): $(OBJDIR)/slablu.o
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $< -lcusolver -lcublas

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB) $(SLIB)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean cxx_test api_timing

CXX_TEST := build/test_leaf_api
cxx_test: $(CXX_TEST)

# Compiled against the reference's own errors.hpp (included first) when it exists.
REF_INC   ?= /root/reference/proj/include
ifneq ($(wildcard $(REF_INC)/hps/errors.hpp),)
CXX_TEST_REF := -I$(REF_INC) -DHPS_TEST_REFERENCE_ERRORS
endif

$(CXX_TEST): tests/cxx/test_leaf_api.cpp include/hps/leaf_gpu.hpp include/hps_leaf_gpu.h $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -Wall -Iinclude $(CXX_TEST_REF) -o $@ $< -L$(dir $(LIB)) -lhps_leaf_b200 \
	    -Wl,-rpath,'$$ORIGIN/../paper_2211_14969_b200/_lib'

API_TIMING := build/api_timing
api_timing: $(API_TIMING)
$(API_TIMING): tools/cxx/api_timing.cpp include/hps/leaf_gpu.hpp include/hps_leaf_gpu.h $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -Iinclude -o $@ $< -L$(dir $(LIB)) -lhps_leaf_b200 \
	    -Wl,-rpath,'$$ORIGIN/../paper_2211_14969_b200/_lib'

# A/B copy of the library with other K2 knobs, e.g.
#   make variant NAME=g128s3 G128_CTAS=3 G128_NSTAGE=3   -> build/variants/g128s3.so
variant:
	$(MAKE) OBJDIR=build/var_$(NAME) LIB=build/variants/$(NAME).so build/variants/$(NAME).so
