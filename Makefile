# Builds the B200 product library (CUDA kernels + C ABI + C++ drop-in API)
# and the CPU checkers under oracle/.  `python -c "import __graft_entry__ as g;
# g.build()"` drives the same targets.
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_2009_07495_b200
BUILD   := build
LIB     := $(PKG)/libigm_b200.so
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -fmad=false -Iinclude
CXXFLAGS:= -O2 -std=c++20 -fPIC -ffp-contract=off -fno-fast-math -Wall -Iinclude
HDRS    := $(wildcard $(PKG)/csrc/*.cuh) $(PKG)/csrc/schedule.hpp $(PKG)/csrc/pencil.hpp include/igm.h $(wildcard include/intgmres/*.hpp)

all: $(LIB) $(BUILD)/e2e_cpp oracle

# the drop-in C++ API timed end to end (bench.py's e2e_cpp leg)
$(BUILD)/e2e_cpp: scripts/e2e_cpp.cpp $(LIB) $(wildcard include/intgmres/*.hpp)
	@mkdir -p $(BUILD)
	g++ -std=c++20 -O2 -Iinclude scripts/e2e_cpp.cpp -L$(PKG) -ligm_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

$(BUILD)/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/%.o: $(PKG)/csrc/%.cpp $(HDRS) $(PKG)/csrc/schedule.hpp
	@mkdir -p $(BUILD)
	g++ $(CXXFLAGS) -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(BUILD)/kernels.o $(BUILD)/setup.o $(BUILD)/capi.o $(BUILD)/shim.o $(BUILD)/schedule.o $(BUILD)/mm_io.o $(BUILD)/experiment.o $(BUILD)/wl32.o $(BUILD)/trace_order.o
	$(NVCC) $(ARCH) -shared -o $@ $^

oracle:
	$(MAKE) -C oracle all
	@if [ -d /root/reference/proj/core ]; then $(MAKE) -C oracle ref; fi

clean:
	rm -rf $(BUILD) $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
