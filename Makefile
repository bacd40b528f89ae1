# Builds the sm_100a C-ABI library (paper_1412_3510_b200/librpca.so) and the
# CPU oracle (oracle/liboracle.so, test infrastructure only).
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr \
            -Xptxas -warn-spills
SRC_DIR  := paper_1412_3510_b200/csrc
SRCS     := $(wildcard $(SRC_DIR)/*.cu)
OBJS     := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
HDRS     := $(wildcard $(SRC_DIR)/*.cuh) include/rpca.h
LIB      := paper_1412_3510_b200/librpca.so
ORACLE   := oracle/liboracle.so

all: $(LIB) $(ORACLE)

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Iinclude -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

$(ORACLE): oracle/rpca_oracle.c
	gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared -std=gnu99 -o $@ $< -lm

clean:
	rm -rf build $(LIB) $(ORACLE)

.PHONY: all clean
