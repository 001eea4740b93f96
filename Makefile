# Builds the B200 (sm_100a) shared library behind include/kairos_b200.h and
# the test-only oracle (oracle/Makefile).
#
#   make            -> paper_2508_06948_b200/_lib/libkairos_b200.so
#   make oracle     -> oracle/_ref/* (C restatement; reference build when present)
#   make sass       -> dump SASS of the library (inspection)

NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 \
            -Xptxas -warn-spills $(NVFLAGS_EXTRA)
PKG      := paper_2508_06948_b200
SRC      := $(PKG)/csrc
OUT      := $(PKG)/_lib
CU       := kx_abi kx_order kx_dispatch kx_orchestrator kx_engine kx_sortlib kx_accuracy kx_priority kx_profiler \
            kx_trace
CPP      := kx_workload
OBJS     := $(patsubst %,$(OUT)/obj/%.o,$(CU)) $(patsubst %,$(OUT)/obj/%.cpp.o,$(CPP))
CXXFLAGS := -std=c++20 -O2 -ffp-contract=off -fPIC -Wall -Wextra
HDRS     := $(wildcard $(SRC)/*.cuh) include/kairos_b200.h

.PHONY: all oracle sass clean
all: $(OUT)/libkairos_b200.so

$(OUT)/obj/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OUT)/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OUT)/obj/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/libkairos_b200.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle:
	$(MAKE) -C oracle

sass: $(OUT)/libkairos_b200.so
	cuobjdump -sass $< | less

clean:
	rm -rf $(OUT)
