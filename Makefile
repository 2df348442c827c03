# Build of the product library (CUDA sm_100a + C++ host) and of the test
# oracles.  `make` builds everything buildable here; the GPU box only needs
# the prebuilt .so files (they travel with the gpurun snapshot).
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
CC       ?= gcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2507_03509_b200
CSRC     := $(PKG)/csrc
LIB      := $(PKG)/libbpdec.so
OBJDIR   := build/obj

CXXFLAGS := -O3 -std=c++20 -fPIC -Wall -Wextra -I$(CSRC) -Iinclude -I/usr/local/cuda/include
NVFLAGS  := -O3 -std=c++20 $(ARCH) -lineinfo -Xcompiler -fPIC,-Wall -I$(CSRC) -Iinclude \
            -Xptxas -v $(NVFLAGS_EXTRA)

HOST_SRC := $(CSRC)/code.cpp $(CSRC)/c_api.cpp $(CSRC)/devmem.cpp
HOST_OBJ := $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.o,$(HOST_SRC))
CU_OBJ   := $(OBJDIR)/decoder.o $(OBJDIR)/harness.o
HDRS     := $(wildcard $(CSRC)/*.hpp $(CSRC)/*.cuh) include/bpdec.h

.PHONY: all lib oracle ref clean guard
all: lib oracle

lib: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJDIR)/decoder.o: $(CSRC)/decoder.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/ptxas.log || (cat $(OBJDIR)/ptxas.log; false)

$(OBJDIR)/harness.o: $(CSRC)/harness.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/ptxas_harness.log || (cat $(OBJDIR)/ptxas_harness.log; false)

$(LIB): $(HOST_OBJ) $(CU_OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread

# oracle/ : CPU restatement (always) + the reference itself (when mounted)
oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

# C++ host-layer test program (reference-shaped API over the C ABI)
COMPAT_TEST := build/compat_test
$(COMPAT_TEST): tests/cpp/compat_test.cpp include/bpdec/etdec_compat.hpp include/bpdec.h $(LIB)
	@mkdir -p build
	$(CXX) -O2 -std=c++20 -Wall -Wextra -Iinclude -o $@ $< -L$(PKG) -lbpdec -Wl,-rpath,'$$ORIGIN/../$(PKG)'

compat_test: $(COMPAT_TEST)
.PHONY: compat_test

# Guard build (bounds-checking stand-in for compute-sanitizer, which this GPU
# pool does not allow): guard zones + poisoned allocations, verified at the
# end of every C-ABI call (csrc/devmem.hpp).  Tests run against it with
# BPDEC_LIB=paper_2507_03509_b200/libbpdec_guard.so (scripts/guard_tests.sh).
GUARD_LIB := $(PKG)/libbpdec_guard.so
GOBJ      := build/gobj
GUARD_HOST_OBJ := $(patsubst $(CSRC)/%.cpp,$(GOBJ)/%.o,$(HOST_SRC))

$(GOBJ)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(GOBJ)
	$(CXX) $(CXXFLAGS) -DBPDEC_GUARD -c $< -o $@

$(GOBJ)/decoder.o: $(CSRC)/decoder.cu $(HDRS)
	@mkdir -p $(GOBJ)
	$(NVCC) $(NVFLAGS) -DBPDEC_GUARD -c $< -o $@ 2> $(GOBJ)/ptxas.log || (cat $(GOBJ)/ptxas.log; false)

$(GOBJ)/harness.o: $(CSRC)/harness.cu $(HDRS)
	@mkdir -p $(GOBJ)
	$(NVCC) $(NVFLAGS) -DBPDEC_GUARD -c $< -o $@ 2> $(GOBJ)/ptxas_harness.log || (cat $(GOBJ)/ptxas_harness.log; false)

$(GUARD_LIB): $(GUARD_HOST_OBJ) $(GOBJ)/decoder.o $(GOBJ)/harness.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread

guard: $(GUARD_LIB)
